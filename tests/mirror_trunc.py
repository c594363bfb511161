"""Numpy mirror of the truncated-TT kernel (csrc/tq_trunc.cu), used by the CPU tests to pin
the algorithm against the oracle before the CUDA code runs.  Test infrastructure only.

Algorithm:
- one-qubit gates act in place, with no centre move (a single-site unitary keeps every
  isometry, so only the gauge differs from the reference);
- before a two-site gate the orthogonality centre moves to the gate's left site through
  isometric splits;
- the two-site block is split by one-sided Jacobi.  Sigma goes to the thin side, and the
  spectrum is truncated by the reference rule (tt.py:85-115);
- term values use full left/right norm environments plus one window per term.
"""

from __future__ import annotations

import math

import numpy as np


TINY = 1e-280   # column pairs below this inner product are numerically zero (no rotation)


def jacobi_cols(x: np.ndarray, tol: float = 1e-15, max_sweeps: int = 30):
    """Orthogonalise the columns of x by complex Hestenes rotations (cyclic order).
    Returns (x V, V) with V unitary (accumulated rotations)."""
    x = x.astype(complex).copy()
    n = x.shape[1]
    v = np.eye(n, dtype=complex)
    for _ in range(max_sweeps):
        rotated = False
        for p in range(n - 1):
            for q in range(p + 1, n):
                a = float(np.vdot(x[:, p], x[:, p]).real)
                b = float(np.vdot(x[:, q], x[:, q]).real)
                g = np.vdot(x[:, p], x[:, q])
                ag = abs(g)
                if ag <= tol * math.sqrt(a) * math.sqrt(b) or ag < TINY:
                    continue
                rotated = True
                e = complex(g.real / ag, g.imag / ag)
                zeta = (b - a) / (2.0 * ag)
                if abs(zeta) > 1e100:
                    t = 0.5 / zeta
                else:
                    t = (1.0 if zeta >= 0 else -1.0) / (abs(zeta) + math.sqrt(1.0 + zeta * zeta))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = c * t
                xp, xq = x[:, p].copy(), x[:, q].copy()
                x[:, p] = c * xp - s * np.conj(e) * xq
                x[:, q] = s * e * xp + c * xq
                vp, vq = v[:, p].copy(), v[:, q].copy()
                v[:, p] = c * vp - s * np.conj(e) * vq
                v[:, q] = s * e * vp + c * vq
        if not rotated:
            break
    return x, v


def keep_rule(s, eps, chi_max):
    """Reference tt.py:85-100 on a descending spectrum."""
    total = float(s @ s)
    k = len(s)
    if eps > 0.0 and s[0] > 0.0:
        k = max(1, int(np.count_nonzero(s > eps * s[0])))
    if chi_max is not None:
        k = min(k, int(chi_max))
    kept = float(s[:k] @ s[:k])
    if total <= 0.0:
        return max(k, 1), 0.0, 1.0
    return k, max(0.0, 1.0 - kept / total), (math.sqrt(total / kept) if kept > 0 else 1.0)


def split_left_iso(m: np.ndarray, eps=0.0, chi_max=None, truncate=False):
    """m = W S with W (rows x k) isometric, rows of S orthogonal (norms sigma, descending)."""
    y, w = jacobi_cols(m.conj().T)           # m^H W = Y  ->  W^H m = Y^H
    sig = np.linalg.norm(y, axis=0)
    order = np.argsort(-sig, kind="stable")
    sig, w = sig[order], w[:, order]
    r = min(m.shape)
    sig = sig[:r]
    if truncate:
        k, disc, scale = keep_rule(sig, eps, chi_max)
    else:
        k, disc, scale = r, 0.0, 1.0
    left = w[:, :k]
    right = (left.conj().T @ m) * scale
    return left, right, disc


def split_right_iso(m: np.ndarray, eps=0.0, chi_max=None, truncate=False):
    """m = L Q with rows of Q orthonormal, columns of L orthogonal (norms sigma, descending)."""
    y, v = jacobi_cols(m)                    # m V = Y  ->  m = Y V^H
    sig = np.linalg.norm(y, axis=0)
    order = np.argsort(-sig, kind="stable")
    sig, v, y = sig[order], v[:, order], y[:, order]
    r = min(m.shape)
    sig = sig[:r]
    if truncate:
        k, disc, scale = keep_rule(sig, eps, chi_max)
    else:
        k, disc, scale = r, 0.0, 1.0
    return y[:, :k] * scale, v[:, :k].conj().T, disc


def simulate(n, gates, eps, chi_max):
    """gates: list of (matrix, sites) with sites (k,) or (i, i+1) on adjacent sites, matrix
    axes in site order (the host expands SWAP chains and flips)."""
    cores = []
    for _ in range(n):
        c = np.zeros((1, 2, 1), dtype=complex)
        c[0, 0, 0] = 1.0
        cores.append(c)
    center = 0
    disc = 0.0
    for mat, sites in gates:
        if len(sites) == 1:
            k = sites[0]
            cores[k] = np.einsum("st,atb->asb", mat, cores[k])
            continue
        i = sites[0]
        while center < i:
            cl, _, cr = cores[center].shape
            q, r, _ = split_left_iso(cores[center].reshape(cl * 2, cr))
            cores[center] = q.reshape(cl, 2, q.shape[1])
            cores[center + 1] = np.tensordot(r, cores[center + 1], axes=([1], [0]))
            center += 1
        while center > i:
            cl, _, cr = cores[center].shape
            l, q, _ = split_right_iso(cores[center].reshape(cl, 2 * cr))
            cores[center] = q.reshape(q.shape[0], 2, cr)
            cores[center - 1] = np.tensordot(cores[center - 1], l, axes=([2], [0]))
            center -= 1
        th = np.tensordot(cores[i], cores[i + 1], axes=([2], [0]))
        th = np.tensordot(mat.reshape(2, 2, 2, 2), th, axes=([2, 3], [1, 2])).transpose(2, 0, 1, 3)
        cl, _, _, cr = th.shape
        mm = th.reshape(cl * 2, 2 * cr)
        if mm.shape[0] <= mm.shape[1]:
            left, right, d = split_left_iso(mm, eps, chi_max, truncate=True)
            center = i + 1
        else:
            left, right, d = split_right_iso(mm, eps, chi_max, truncate=True)
            center = i
        k = left.shape[1]
        cores[i] = left.reshape(cl, 2, k)
        cores[i + 1] = right.reshape(k, 2, cr)
        disc += d
    return cores, disc


PAULI = {"X": np.array([[0, 1], [1, 0]], complex), "Y": np.array([[0, -1j], [1j, 0]]),
         "Z": np.array([[1, 0], [0, -1]], complex)}
PAULI.update({1: PAULI["X"], 2: PAULI["Y"], 3: PAULI["Z"]})


def term_values(cores, terms):
    """<psi|P_t|psi> from full norm environments (empty term -> 1, as the reference)."""
    n = len(cores)
    L = [np.ones((1, 1), complex)]
    for k in range(n):
        a = cores[k]
        L.append(np.einsum("ab,asc,bsd->cd", L[-1], a.conj(), a))
    R = [None] * (n + 1)
    R[n] = np.ones((1, 1), complex)
    for k in range(n - 1, -1, -1):
        a = cores[k]
        R[k] = np.einsum("asc,cd,bsd->ab", a.conj(), R[k + 1], a)
    out = np.zeros(len(terms), complex)
    for t, (_, ops) in enumerate(terms):
        ops = dict(ops)
        if not ops:
            out[t] = 1.0
            continue
        lo, hi = min(ops), max(ops)
        x = L[lo]
        for k in range(lo, hi + 1):
            a = cores[k]
            p = PAULI[ops[k]] if k in ops else np.eye(2)
            x = np.einsum("ab,asc,st,btd->cd", x, a.conj(), p, a)
        out[t] = np.einsum("ab,ab->", x, R[hi + 1])
    return out
