import sys; import os; R=os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0,R); sys.path.insert(0,os.path.join(R,"tests"))
import numpy as np
import oracle as O
from paper_2112_10239_b200 import truncated as TR, chain as C
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets
from paper_2112_10239_b200.hamiltonians import tfim
c = layered_circuit(12, 12, "ry", "cnot")
terms = C.normalize_terms(tfim(12)); oterms = O.tfim_terms(12)
th = theta_sets(c.n_params, 3, seed=7)
for eps, chi in ((0.0, 4), (1e-3, None), (1e-2, 6)):
    for dt in ("complex128","complex64"):
        r = TR.simulate_terms(c, terms, th, eps, chi, dtype=dt)
        tt = O.simulate_tt(O.OCircuit(12, [(g.name, tuple(g.wires), g.param) for g in c.gates], list(c.trainable)), th[0], eps=eps, chi_max=chi)
        ov = O.tt_term_values(tt, oterms)
        print(eps, chi, dt, "dv %.2e"%np.max(np.abs(r.values[0]-ov)), "disc", r.discarded[0], tt.discarded, list(r.bonds[0]), list(tt.bonds))
