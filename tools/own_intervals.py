"""Bucket-interval jobs on one GPU, own-bucket layout vs the plain filter
(dev tool): per interval of a K-way split, device time of create + run, the
job's planned terms and entries. Usage: python tools/own_intervals.py c2 8 [kappa]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1210_0461_b200 as crop  # noqa: E402
from paper_1210_0461_b200 import _native as nat  # noqa: E402
from paper_1210_0461_b200 import kernels, workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kappa = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.kappa
only = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else None
dtx = workloads.generate_pairs_workload(cfg)
h = crop.make_hashes(crop.HashConfig(kappa, crop.derive_seed(0, "instance:0")))
tab = kernels.hash_tables(h, cfg.n_items)
flush = torch.empty(1 << 28, dtype=torch.int32, device="cuda")


def timed(fn, reps=4):
    best = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1))
    best.sort()
    return best[len(best) // 2], out


def whole():
    job = kernels.PairCountJob(dtx, True, None, keep=tab)
    ent = job.run()
    job.close()
    return ent.n, job.total_terms, False


t, (n, terms, _) = timed(whole)
print(f"{cfg.name}: whole job {t:.3f} ms, {terms} terms, {n} entries", flush=True)
tot = 0
for w, a in enumerate(crop.WorkerAssignment.split(kappa, K)):
    if only is not None and w not in only:
        continue
    iv = kernels.interval_struct(kappa, a.start, a.stop, *tab)
    for flags in (0, nat.PAIRS_NO_OWN):
        def one():
            job = kernels.PairCountJob(dtx, True, iv, keep=tab, flags=flags)
            job.set_timing(True)
            ent = job.run()
            ph = job.phase_ms()
            job.close()
            return ent.n, job.total_terms, job.own, ph
        t, (n, terms, own, ph) = timed(one)
        if flags == 0:
            tot += terms
        print(f"  interval {w} [{a.start},{a.stop}) {'own ' if own else 'plain'}: {t:.3f} ms "
              f"terms={terms} entries={n} write={ph['write']:.3f} count={ph['count']:.3f}",
              flush=True)
print(f"sum of own terms {tot}")
