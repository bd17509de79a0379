"""Time one rank's share of a G-GPU run on one GPU (bucket interval filter) (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = workloads.CONFIGS[name]
dtx = workloads.generate_pairs_workload(cfg)
config = crop.EngineConfig(kappa=cfg.kappa, ss_capacity=2 ** 31, workers=cfg.workers, cs_enabled=False, seed=0)
h = crop.make_hashes(crop.HashConfig(cfg.kappa, config.instance_seeds()[0]))
tab = kernels.hash_tables(h, cfg.n_items)
mode = sys.argv[3] if len(sys.argv) > 3 else "tiles"
for r in range(min(G, 2)):
    asg = crop.WorkerAssignment.split(cfg.kappa, G)[r]
    iv = kernels.interval_struct(cfg.kappa, asg.start, asg.stop, *tab) if mode == "buckets" else None
    shard = (r, G) if mode == "tiles" else (0, 1)
    for it in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        job = kernels.PairCountJob(dtx, True, iv, keep=tab, shard=shard)
        job.set_timing(True)
        ent = job.run()
        e1.record()
        torch.cuda.synchronize()
        ph = job.phase_ms()
        job.close()
    print(f"{name} G={G} {mode} rank {r}: {e0.elapsed_time(e1):.3f} ms "
          f"entries={ent.n} phases={ {k: round(v, 3) for k, v in ph.items()} }")
