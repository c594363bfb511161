/*
 * tq_trunc.h — C ABI of the truncated tensor-train engine.
 *
 *   tq_tt_simulate  replaces  simulate_tt(circuit, eps, chi_max)        tt.py:237-244
 *                             (apply_gate_tt tt.py:186-234, _apply_adjacent tt.py:168-183,
 *                              _split_matrix / _truncate_spectrum tt.py:85-115,
 *                              _position_center tt.py:146-161)
 *                   followed by the per-term windows of _expval_tt     hamiltonians.py:129-164
 *                   for every theta-set of a batch.
 *
 * Gates come from the host compiler (paper_2112_10239_b200/truncated.py): one- and two-site
 * gates on adjacent sites, SWAP chains already expanded, matrix axes in site order.  A
 * trainable rotation (rot != 0) is evaluated from theta[b][slot] on the device.
 *
 * Per theta-set outputs: values [B][T] (re, im float64) = <psi|P_t|psi> (1 for an empty
 * term, as the reference), discarded [B] (accumulated discarded weight), norm2 [B] (<psi|psi>,
 * optional), bonds [B][n+1]
 * (final bond dimensions), flags [B] (1 when a bond needed more than chi_cap).
 * dtype: TQ_C64 -> theta float32, TQ_C128 -> float64.
 */
#ifndef TQ_TRUNC_H
#define TQ_TRUNC_H

#include <stddef.h>
#include <stdint.h>

#include "tq_engine.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One gate of the expanded TEBD program (truncated.py TGATE_DTYPE, 288 bytes). */
typedef struct {
  int32_t kind;      /* 1: one-site on `site`; 2: two-site on (site, site + 1) */
  int32_t site;
  int32_t rot;       /* 0: constant matrix m; 1 rx, 2 ry, 3 rz, 4 crz from theta[slot] */
  int32_t slot;
  int32_t flip;      /* rot == crz with reversed wires: swap the two tensor legs */
  int32_t pad[3];
  double m[32];      /* 2x2 or 4x4 complex, row-major, (re, im) interleaved */
} tq_tgate;

/* Workspace for `batch` theta-sets of an n-qubit train with bond capacity chi_cap (<= 32). */
size_t tq_tt_workspace_bytes(int n_qubits, int batch, int chi_cap, int dtype);

tq_status tq_tt_simulate(int n_qubits, const void* gates, int n_gates, int dtype, int batch,
                         const void* theta, int64_t theta_stride, double eps, int chi_cap, int chi_max,
                         const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off,
                         const int8_t* codes, int n_terms, void* values, double* discarded,
                         double* norm2, int32_t* bonds, int32_t* flags, void* workspace,
                         size_t workspace_bytes, void* stream);

/* The same engine in phases, over a caller-owned device train (reference TTState, tt.py:38-76):
 * cores [B][n][2 cap^2] complex (core k dense (chi_k, 2, chi_{k+1}) at the start of its slot),
 * bonds [B][n+1], centers [B], discarded [B].
 *   tq_tt_run       simulate_tt(circuit, eps, chi_max)                 tt.py:237-244
 *   tq_tt_compress  compress(tt, eps, chi_max), in place                tt.py:299-320
 *   tq_tt_values    per-term windows + <psi|psi>                        hamiltonians.py:129-164 */
size_t tq_tt_state_bytes(int n_qubits, int batch, int chi_cap, int dtype);
size_t tq_tt_values_workspace_bytes(int n_qubits, int batch, int chi_cap, int dtype);
tq_status tq_tt_run(int n_qubits, const void* gates, int n_gates, int dtype, int batch, const void* theta,
                    int64_t theta_stride, double eps, int chi_cap, int chi_max, void* cores, int32_t* bonds,
                    int32_t* centers, double* discarded, int32_t* flags, void* stream);
tq_status tq_tt_compress(int n_qubits, int dtype, int batch, double eps, int chi_cap, int chi_max, void* cores,
                         int32_t* bonds, int32_t* centers, double* discarded, int32_t* flags, void* stream);
/* apply_gate_tt over a whole circuit on trains the caller already holds (tt.py:186-234): every row
 * continues from its own cores / bonds / centre, discarded weight accumulates. */
tq_status tq_tt_apply(int n_qubits, const void* gates, int n_gates, int dtype, int batch, const void* theta,
                      int64_t theta_stride, double eps, int chi_cap, int chi_max, void* cores, int32_t* bonds,
                      int32_t* centers, double* discarded, int32_t* flags, void* stream);
tq_status tq_tt_values(int n_qubits, int dtype, int batch, int chi_cap, const void* cores, const int32_t* bonds,
                       const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off, const int8_t* codes,
                       int n_terms, void* values, double* norm2, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Straight-through gradient of a truncated run (reference grad_expval with eps > 0 or a binding
 * chi_max: _tt_taped_state autodiff.py:339-363, _tt_taped_split autodiff.py:315-336).  The taped
 * state is built without centre moves; each two-site split keeps its SVD factor U_k (m <= n) or
 * Vh_k as a constant and the other factor as the differentiable projection.
 *   tq_tt_taped   runs that construction for B theta-sets, writes the per-term values of the
 *                 final train (an empty term gives <psi|psi>, as the tape) and records every
 *                 split's constant factor + (k, side, rescale) into `tape`
 *                 (tq_tt_tape_bytes(n_two_site, B, cap, dtype) bytes);
 *   tq_tt_replay  re-runs it for `rows` angle sets with the constants of the recorded theta-set
 *                 parent[row] frozen (no SVD).  With the constants frozen each angle enters as
 *                 c + a cos(t/2) + b sin(t/2), so the shift rule on replayed values is the exact
 *                 straight-through derivative.
 * n_two_site = number of kind-2 rows of the gate table (the tape slots per theta-set). */
size_t tq_tt_tape_bytes(int n_two_site, int batch, int chi_cap, int dtype);
tq_status tq_tt_taped(int n_qubits, const void* gates, int n_gates, int n_two_site, int dtype, int batch,
                      const void* theta, int64_t theta_stride, double eps, int chi_cap, int chi_max,
                      const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off, const int8_t* codes,
                      int n_terms, void* values, double* norm2, int32_t* bonds, int32_t* flags, void* tape,
                      const void* init_cores, const int32_t* init_bonds,
                      void* workspace, size_t workspace_bytes, void* stream);
tq_status tq_tt_replay(int n_qubits, const void* gates, int n_gates, int n_two_site, int dtype, int rows,
                       const void* theta, int64_t theta_stride, int chi_cap, const int32_t* parent, int tape_batch,
                       const void* tape, const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off,
                       const int8_t* codes, int n_terms, void* values, double* norm2, int32_t* bonds, int32_t* flags,
                       const void* init_cores, const int32_t* init_bonds,
                       void* workspace, size_t workspace_bytes, void* stream);
/* init_cores / init_bonds (optional, may be NULL): an input train (reference TTState, tt.py:38-76)
 * in the slot layout [n][2 cap^2] with bonds [n+1], shared by every row: the circuit then runs on
 * that state instead of |0...0>.  With eps = 0 and no binding chi_max every split keeps a square
 * unitary factor, so the replayed shift rule is the EXACT gradient of <state|U^H H U|state>
 * (autodiff.py:8-13): the differentiable path for arbitrary input trains. */

/* <a_r|b_r> for every row r of two batches of trains (slot layout, bonds [B][n+1]); out [B] complex
 * (re, im float64), a conjugated: the reference's tt_inner (tt.py:247-255) on arbitrary trains. */
tq_status tq_tt_inner(int n_qubits, int dtype, int batch, int chi_cap, const void* cores_a, const int32_t* bonds_a,
                      const void* cores_b, const int32_t* bonds_b, void* out, void* stream);

/* Measured FP64 FMA throughput of this GPU (the roofline denominator of the complex128 path). */
tq_status tq_tt_dfma_peak(int32_t iters, void* stream, double* tflops_out);

#ifdef __cplusplus
}
#endif

#endif /* TQ_TRUNC_H */
