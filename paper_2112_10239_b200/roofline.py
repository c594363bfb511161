"""Algorithmic work model of the engine's sweeps (DESIGN.md section "Roofline").

Counts complex multiply-adds (cMAC, 8 real flops each) exactly as the kernels issue
them for an UNSEGMENTED chain (segments=1), so light-cone halo redundancy never
inflates ``achieved``:

  fold        chi_l*chi_r pairs x ops x 4 cMAC                       (both sweeps)
  RL          N: 2*Db*chi_l*chi_r^2     P: 2*Da*chi_l^2*chi_r x h(chi_l)
  LR          M: 2*Da*chi_l^2*chi_r     Lam: 2*Db*chi_r^2*chi_l x h(chi_r)     G: 2*Db*chi_l*chi_r^2
              (h = herm_fraction: the Hermitian transfers' upper-tile share, 1 below chi 16)
  adjoint     chi_l*chi_r pairs x ops x 12 cMAC (u and v walks + sigma contraction)
  brackets    2*D*chi_l*chi_r x (edges per channel) cMAC (counted)

HBM bytes per evaluation (compulsory): theta (P reals) + gradient (P reals) + energy
(16 B) + the stored right environments written once by RL and read once by LR.
"""

from __future__ import annotations

import numpy as np


def herm_fraction(n) -> np.ndarray:
    """Share of an n x n environment transfer the Hermitian GEMM path computes (n >= 16:
    4x2 tiles of the upper triangle, tq_engine.cu gemm_group HERM; 72 of 128 tiles at 32)."""
    n = np.asarray(n, dtype=np.float64)
    nb, nc = n / 4, n / 2
    frac = (nb * nc - nb * (nb - 1)) / np.maximum(nb * nc, 1)
    return np.where(n >= 16, frac, 1.0)


def sweep_cmacs(plan) -> dict:
    """cMACs per theta-set: 'rl' right-to-left sweep, 'lr' left-to-right sweep (gradient
    mode with the column adjoint, or values mode with the rho contractions)."""
    s = plan.sites
    cl = s["chi_l"].astype(np.float64)
    cr = s["chi_r"].astype(np.float64)
    nops = s["op_count"].astype(np.float64)
    pairs = cl * cr
    fold = pairs * nops * 4
    # energy mode: the P (RL) and Lambda (LR) transfers are Hermitian, computed on upper tiles
    hp = herm_fraction(cl) if plan.mode != "values" else 1.0
    hl = herm_fraction(cr)
    rl = 2 * s["rl_db"] * cl * cr * cr + 2 * s["rl_da"] * cl * cl * cr * hp + 2 * s["rl_edge_count"] * cl * cr
    lr = (2 * s["lr_da"] * cl * cl * cr + 2 * s["lr_db"] * cr * cr * cl * hl + 2 * s["lr_db"] * cl * cr * cr
          + 2 * s["lr_edge_count"] * cl * cr)
    if plan.mode == "values":
        lr = (2 * s["lr_da"] * cl * cl * cr + 2 * s["lr_db"] * cr * cr * cl + 2 * s["lr_da"] * cl * cr * cr
              + 4 * s["lr_da"] * cl * cr * (s["fin_count"] > 0) + 2 * s["lr_edge_count"] * cl * cr)
        adj = np.zeros_like(fold)
    else:
        # column adjoint counted on the digit tree (the minimal walk): per tree entry one
        # forward matvec (4), one backward matvec (4), the digit reduction (~2) and the
        # sigma contraction (2)
        ops = plan.ops
        adj = np.zeros_like(fold)
        for i in range(len(s)):
            b, c = int(s["op_begin"][i]), int(s["op_count"][i])
            if c:
                last = ops[b + c - 1]
                entries = int(last["tbase"]) + (1 << (int(last["toff"]) + int(last["bits"])))
                adj[i] = 12.0 * entries
    # the left-to-right sweep reloads the folded cores stored by the right-to-left sweep
    return {"rl": float(np.sum(fold + rl)), "lr": float(np.sum(lr)), "adj": float(np.sum(adj)),
            "fold": float(np.sum(fold)), "adjoint": float(np.sum(adj))}


def env_bytes(plan, real_bytes: int = 4) -> float:
    """Stored right-environment bytes for one theta-set (written once, read once)."""
    return float(plan.env_total) * 2 * real_bytes


def eval_model(plan, grad: bool = True, real_bytes: int = 4, real: bool = False) -> dict:
    """Per-evaluation (one theta-set) flops and compulsory HBM bytes.

    ``real``: the plan runs the engine's real-path instantiation (tq_chain.real_path,
    complex64 energy mode; chain.real_path): every operand's imaginary part is an exact
    zero and the sweeps issue one real FMA (2 flops) per cMAC instead of 8 flops; the column
    adjoint's real instantiation exists for the digit-tree layout only (chi_max >= 16,
    tq_engine.cu make_adj_layout), the chi <= 8 warp adjoint stays complex."""
    c = sweep_cmacs(plan)
    per = 2.0 if real else 8.0
    per_adj = 2.0 if real and plan.chi_max >= 16 else 8.0
    flops_rl = per * c["rl"]
    flops_lr = per * c["lr"] if grad else 0.0
    flops_adj = per_adj * c["adj"] if grad else 0.0
    P = plan.n_params
    byts = P * real_bytes + 16
    if grad:
        byts += P * real_bytes + 2 * env_bytes(plan, real_bytes)
    return {"flops_rl": flops_rl, "flops_lr": flops_lr, "flops_adj": flops_adj,
            "flops": flops_rl + flops_lr + flops_adj, "bytes": byts, "cmacs": c,
            "flops_per_cmac": per, "flops_per_cmac_adj": per_adj, "real_path": bool(real)}


def survey_model(plan, n_terms_1: int, n_terms_2: int, layers: int, grad: bool = True) -> dict:
    """SURVEY.md section 8(d)'s official per-evaluation work (the judge's formulas).

    ``plan`` must be the UNSEGMENTED plan (segments=1) so its sites carry the bonds
    chi_k = 2^{c_k} of the factored chain (chi_0 = chi_n = 1).  Per site k:
      step_k = 2 chi_k chi_{k+1} (chi_k + chi_{k+1}) cMAC   (one transfer sum_s A_s^H E A_s)
      fold_k = 4 L chi_k chi_{k+1} cMAC                     (L = rows + lines)
      F_fwd  = 8 [sum fold + 2 sum step + (T1 + 2 T2) mean(step)]   real flops
      F_eval = 3 F_fwd with the gradient, F_fwd forward-only
      B_eval = 4P + 4P + 4 + 16 sum_k chi_k^2 bytes (gradient), 4P + 4 forward-only."""
    s = plan.sites
    cl = s["chi_l"].astype(np.float64)
    cr = s["chi_r"].astype(np.float64)
    step = 2 * cl * cr * (cl + cr)
    fold = 4 * layers * cl * cr
    f_fwd = 8 * (fold.sum() + 2 * step.sum() + (n_terms_1 + 2 * n_terms_2) * step.mean())
    P = plan.n_params
    if grad:
        chi2 = float(np.sum(cr[:-1] ** 2)) if len(cr) > 1 else 0.0   # cuts 1..n-1
        byts = 4 * P + 4 * P + 4 + 16 * chi2
    else:
        byts = 4 * P + 4
    return {"F_fwd": float(f_fwd), "F_eval": float(3 * f_fwd if grad else f_fwd), "B_eval": float(byts)}
