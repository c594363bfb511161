"""numpy complex128 mirror of the CUDA kernels — test infrastructure.

Executes a ChainPlan exactly the way ``csrc/tq_engine.cu`` does (column fold,
right-to-left MPO sweep, left-to-right gradient sweep with the per-pair fold
adjoint, value finalisation), so the compiler's tables and the hand-derived
adjoint can be validated on the CPU against the oracle before any kernel runs.
"""

from __future__ import annotations

import numpy as np

from paper_2112_10239_b200 import chain as C

SIGMA = {C.KIND_RX: np.array([[0, 1], [1, 0]], complex),
         C.KIND_RY: np.array([[0, -1j], [1j, 0]], complex),
         C.KIND_RZ: np.array([[1, 0], [0, -1]], complex)}
OPM = {0: np.eye(2, dtype=complex), 1: np.array([[0, 1], [1, 0]], complex),
       2: np.array([[0, -1j], [1j, 0]], complex), 3: np.diag([1, -1]).astype(complex)}


def _mat(rec, theta):
    if rec["kind"] == C.KIND_CONST:
        m = rec["m"]
        return np.array([m[0] + 1j * m[1], m[2] + 1j * m[3], m[4] + 1j * m[5], m[6] + 1j * m[7]]).reshape(2, 2)
    t = float(theta[rec["slot"]]) if rec["slot"] >= 0 else float(rec["angle"])
    c, s = np.cos(t / 2), np.sin(t / 2)
    return c * np.eye(2) - 1j * s * SIGMA[int(rec["kind"])]


def site_ops(plan, site, theta):
    """Per op: (src, shift, mask, [matrix per digit], [kind per digit], tidx)."""
    out = []
    for o in plan.ops[site["op_begin"]: site["op_begin"] + site["op_count"]]:
        nd = 1 << int(o["bits"])
        recs = [plan.mats[int(o["mat"]) + d] for d in range(nd)]
        out.append((int(o["src"]), int(o["shift"]), nd - 1, [_mat(r, theta) for r in recs],
                    [int(r["kind"]) for r in recs], int(o["tidx"])))
    return out


def _digits(src, shift, mask, al, be):
    if src == C.SRC_ALPHA:
        return (al >> shift) & mask
    if src == C.SRC_BETA:
        return (be >> shift) & mask
    return np.zeros_like(al)


def fold(plan, site, theta, keep=False):
    cl, cr = int(site["chi_l"]), int(site["chi_r"])
    al, be = np.meshgrid(np.arange(cl), np.arange(cr), indexing="ij")
    init = site["init"]
    v = np.zeros((cl, cr, 2), complex)
    v[..., 0] = init[0] + 1j * init[1]
    v[..., 1] = init[2] + 1j * init[3]
    hist = [v]
    ops = site_ops(plan, site, theta)
    for src, shift, mask, mats, kinds, _ in ops:
        d = _digits(src, shift, mask, al, be)
        M = np.stack(mats)[d]                      # (cl, cr, 2, 2)
        v = np.einsum("abij,abj->abi", M, v)
        hist.append(v)
    ok = np.ones((cl, cr), bool)
    for p in plan.passes[site["pass_begin"]: site["pass_begin"] + site["pass_count"]]:
        m = (1 << int(p["bits"])) - 1
        ok &= ((al >> int(p["sa"])) & m) == ((be >> int(p["sb"])) & m)
    A = np.where(ok[..., None], v, 0).transpose(2, 0, 1)  # (2, cl, cr)
    if keep:
        return A, hist, ops, ok, al, be
    return A


def _apply_edges(edges, srcs, nsrc_shape):
    """bracket[b][s'] = sum_edges coef * sum_s O_{s's} src[a][s]  (edges: (a,b,op,c))."""
    out = {}
    for a, b, op, c in edges:
        O = OPM[op]
        for sp in range(2):
            acc = out.setdefault((b, sp), np.zeros(nsrc_shape, complex))
            for s in range(2):
                if O[sp, s] != 0:
                    acc += c * O[sp, s] * srcs[a][s]
    return out


def _edges(plan, site, which, coef):
    b0 = int(site[f"{which}_edge_begin"])
    res = []
    for e in plan.edges[b0: b0 + int(site[f"{which}_edge_count"])]:
        c = 1.0 if e["coef"] < 0 else coef[int(e["coef"])]
        res.append((int(e["a"]), int(e["b"]), int(e["op"]), c))
    return res


def rl_pass(plan, seg, theta, coef):
    """Right-to-left MPO sweep; returns (P^START at the left boundary, stored envs per local cut)."""
    sb, nsite = int(seg["site_begin"]), int(seg["site_count"])
    P = {0: np.ones((1, 1), complex)}  # channel -> matrix at the current right cut
    envs = {nsite: P}
    for q in range(nsite - 1, -1, -1):
        site = plan.sites[sb + q]
        A = fold(plan, site, theta)
        N = {b: [A[s] @ P[b] for s in range(2)] for b in P}
        cl, cr = A.shape[1], A.shape[2]
        # edges a(left)<-b(right): bracket'[a][s'] = sum coef sum_s O_{s's} N[b][s]
        rev = [(b, a, op, c) for a, b, op, c in _edges(plan, site, "rl", coef)]
        br = _apply_edges(rev, N, (cl, cr))
        newP = {}
        for a in range(int(site["rl_da"])):
            acc = np.zeros((cl, cl), complex)
            for sp in range(2):
                if (a, sp) in br:
                    acc += br[(a, sp)] @ A[sp].conj().T
            newP[a] = acc
        P = newP
        envs[q] = P
    return P[0][0, 0], envs


def lr_grad(plan, seg, theta, coef, envs):
    """Left-to-right sweep with G and the per-pair fold adjoint; returns local grads."""
    sb, nsite = int(seg["site_begin"]), int(seg["site_count"])
    gl = np.zeros(int(seg["gslot_count"]))
    Lam = {0: np.ones((1, 1), complex)}
    for q in range(nsite):
        site = plan.sites[sb + q]
        A, hist, ops, ok, al, be = fold(plan, site, theta, keep=True)
        cl, cr = A.shape[1], A.shape[2]
        M = {a: [Lam[a] @ A[s] for s in range(2)] for a in Lam}
        br = _apply_edges(_edges(plan, site, "lr", coef), M, (cl, cr))
        Pn = envs[q + 1]
        G = [np.zeros((cl, cr), complex) for _ in range(2)]
        newL = {}
        for b in range(int(site["lr_db"])):
            accL = np.zeros((cr, cr), complex)
            for sp in range(2):
                if (b, sp) in br:
                    accL += A[sp].conj().T @ br[(b, sp)]
                    G[sp] += br[(b, sp)] @ Pn[b]
            newL[b] = accL
        Lam = newL
        # fold adjoint: contributions Im<u_l, sigma v_l> per trainable op
        g = np.stack([np.where(ok, G[0], 0), np.where(ok, G[1], 0)], axis=-1)  # (cl, cr, 2)
        u = g
        for l in range(len(ops) - 1, -1, -1):
            src, shift, mask, mats, kinds, tidx = ops[l]
            d = _digits(src, shift, mask, al, be)
            Ms = np.stack(mats)[d]
            kd = np.array(kinds)[d]
            v = hist[l + 1]
            if tidx >= 0:
                tot = 0.0
                for k, sig in SIGMA.items():
                    sel = kd == k
                    if sel.any():
                        sv = np.einsum("ij,abj->abi", sig, v)
                        tot += np.sum(np.where(sel, np.einsum("abi,abi->ab", u.conj(), sv), 0)).imag
                o = plan.ops[int(site["op_begin"]) + l]
                gl[int(o["gidx"])] += tot
            u = np.einsum("abji,abj->abi", Ms.conj(), u)
    return gl


def lr_values(plan, seg, theta, envs, T):
    sb, nsite = int(seg["site_begin"]), int(seg["site_count"])
    out = {}
    Lam = {0: np.ones((1, 1), complex)}
    for q in range(nsite):
        site = plan.sites[sb + q]
        A = fold(plan, site, theta)
        cl, cr = A.shape[1], A.shape[2]
        M = {a: [Lam[a] @ A[s] for s in range(2)] for a in Lam}
        R = envs[q + 1][0]
        for f in plan.fins[site["fin_begin"]: site["fin_begin"] + site["fin_count"]]:
            a, t, op = int(f["a"]), int(f["b"]), int(f["op"])
            O = OPM[op]
            val = 0j
            for sp in range(2):
                for s in range(2):
                    if O[sp, s] != 0:
                        val += O[sp, s] * np.sum(A[sp].conj() * (M[a][s] @ R))
            out[t] = val
        br = _apply_edges(_edges(plan, site, "lr", np.ones(T)), M, (cl, cr))
        newL = {}
        for b in range(int(site["lr_db"])):
            acc = np.zeros((cr, cr), complex)
            for sp in range(2):
                if (b, sp) in br:
                    acc += A[sp].conj().T @ br[(b, sp)]
            newL[b] = acc
        Lam = newL
    return out


def energy_grad(plan, theta, coef):
    """Full E (complex) and dE/dtheta via the mirror."""
    E = complex(plan.e_const)
    partial = np.zeros(plan.n_gslots)
    for seg in plan.segs:
        e, envs = rl_pass(plan, seg, theta, coef)
        E += e
        gl = lr_grad(plan, seg, theta, coef, envs)
        partial[int(seg["gslot_begin"]): int(seg["gslot_begin"]) + len(gl)] = gl
    grad = np.array([partial[plan.gred_idx[plan.gred_ptr[p]: plan.gred_ptr[p + 1]]].sum()
                     for p in range(plan.n_params)])
    return E, grad


def term_values(plan, theta):
    vals = np.where(plan.term_active == 0, 1.0 + 0j, 0j).astype(complex)
    for seg in plan.segs:
        _, envs = rl_pass(plan, seg, theta, np.ones(plan.n_terms))
        for t, v in lr_values(plan, seg, theta, envs, plan.n_terms).items():
            vals[t] = v
    return vals
