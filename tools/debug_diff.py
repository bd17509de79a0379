import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
from paper_1210_0461_b200 import kernels, workloads
name = sys.argv[1]; n_tx = int(sys.argv[2])
cfg = workloads.CONFIGS[name]
dtx = workloads.generate_pairs_workload(cfg, n_tx=n_tx)
off, items = dtx.to_host()
job = kernels.PairCountJob(dtx, True, None)
print("tiles", job.n_tiles, "units", job.n_units)
ent = job.run()
r, c, w = ent.to_numpy()
orow, ocol, ow = oracle.pair_supports(off, items)
g = {(int(a), int(b)): int(x) for a, b, x in zip(r, c, w)}
o = {(int(a), int(b)): int(x) for a, b, x in zip(orow, ocol, ow)}
extra = [k for k in g if k not in o]
missing = [k for k in o if k not in g]
diff = [k for k in o if k in g and g[k] != o[k]]
print("gpu", len(g), "oracle", len(o), "extra", len(extra), "missing", len(missing), "diff", len(diff))
print("extra sample", extra[:10], [g[k] for k in extra[:10]])
print("missing sample", missing[:10], [o[k] for k in missing[:10]])
print("diff sample", [(k, g[k], o[k]) for k in diff[:10]])
dup = len(r) - len(g)
print("duplicate keys in gpu output", dup)
import collections
print("rows of extra", collections.Counter(k[0] for k in extra).most_common(10))
print("rows of diff", collections.Counter(k[0] for k in diff).most_common(10))
