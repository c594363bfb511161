cat > /tmp/one.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2112_10239_b200 import truncated as TR, chain as C
from paper_2112_10239_b200.report import tfim_workload
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import theta_sets
c = tfim_workload(100, 3000); terms = C.normalize_terms(tfim(100))
TR.simulate_terms(c, terms, theta_sets(c.n_params, 1, seed=0), 0.0, 32)
PY
ncu --set full --import-source on --clock-control none -k regex:tt_simulate -c 1 -f -o /tmp/tt32 python /tmp/one.py > /dev/null 2>&1
python tools/ncu_summary.py /tmp/tt32.ncu-rep > gpurun_out/ncu_tt32.txt 2>&1
python tools/ncu_lines.py /tmp/tt32.ncu-rep tt_simulate paper_2112_10239_b200/libtq_engine.so 40 >> gpurun_out/ncu_tt32.txt 2>&1
