import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1210_0461_b200 import kernels, workloads
cfg = workloads.CONFIGS["c2"]
dtx = workloads.generate_pairs_workload(cfg, n_tx=2000)
ent = kernels.count_pairs(dtx, True)
print("n", ent.n)
