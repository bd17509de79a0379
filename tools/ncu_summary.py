"""Summarise an `ncu --set full` report of the counting path into
profiles/ncu_summary.json (per-kernel duration, DRAM bytes, L2 hit rate,
issue utilisation) and print a table (dev tool)."""
import csv
import io
import json
import subprocess
import sys

rep, config = sys.argv[1], sys.argv[2]
out_json = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_summary.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = {"gpu__time_duration.sum": "ms", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "lts__t_sector_hit_rate.pct": "l2_hit_pct", "smsp__inst_executed.sum": "warp_instructions",
        "smsp__inst_executed_op_shared_atom.sum": "smem_atom_inst",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum": "smem_atom_wavefronts",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum": "smem_atom_bank_conflicts",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
        "lts__t_sectors_op_atom.sum": "l2_atom_sectors", "lts__t_sectors_op_red.sum": "l2_red_sectors",
        "sm__cycles_elapsed.avg": "sm_cycles",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "launch__registers_per_thread": "registers", "launch__grid_size": "grid", "launch__block_size": "block"}
units = rows[1]
kernels = {}
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    rec = {}
    for m, k in want.items():
        if m not in d:
            continue
        try:
            v = float(d[m].replace(",", ""))
        except ValueError:
            continue
        if v != v:  # n/a
            continue
        u = units[h.index(m)]
        if k == "ms":
            v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                  "second": 1e3, "s": 1e3}.get(u, 1.0)
        if k.startswith("dram"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
                  "GB": 1e9}.get(u, 1.0)
        rec[k] = v
    kernels.setdefault(name, []).append(rec)
summary = {}
tot_ms = sum(x["ms"] for v in kernels.values() for x in v)
path = 0.0
print(f"{'kernel':32s} {'n':>2s} {'ms':>8s} {'share':>6s} {'DRAM rd GB':>10s} {'DRAM wr GB':>10s} {'L2 hit':>6s} {'issue%':>6s}")
for name, v in sorted(kernels.items(), key=lambda kv: -sum(x["ms"] for x in kv[1])):
    n = len(v)
    keys = set().union(*v)
    agg = {k: sum(x.get(k, 0.0) for x in v) / n for k in keys}
    agg.setdefault("dram_read", 0.0)
    agg.setdefault("dram_write", 0.0)
    agg.setdefault("ms", 0.0)
    summary[name] = {"launches": n, "ms_per_launch": round(agg["ms"], 4),
                     "dram_bytes_per_launch": int(agg["dram_read"] + agg["dram_write"]),
                     "dram_read_bytes": int(agg["dram_read"]), "dram_write_bytes": int(agg["dram_write"]),
                     "l2_hit_pct": round(agg.get("l2_hit_pct", 0), 1),
                     "issue_active_pct": round(agg.get("issue_active_pct", 0), 1),
                     "occupancy_pct": round(agg.get("occupancy_pct", 0), 1),
                     "warp_instructions": int(agg.get("warp_instructions", 0)),
                     "smem_atom_inst": int(agg.get("smem_atom_inst", 0)),
                     "smem_atom_wavefronts": int(agg.get("smem_atom_wavefronts", 0)),
                     "smem_atom_bank_conflicts": int(agg.get("smem_atom_bank_conflicts", 0)),
                     "smem_bank_conflicts": int(agg.get("smem_bank_conflicts", 0)),
                     "l2_atom_sectors": int(agg.get("l2_atom_sectors", 0)),
                     "l2_red_sectors": int(agg.get("l2_red_sectors", 0)),
                     "sm_cycles": int(agg.get("sm_cycles", 0)),
                     "registers": int(agg.get("registers", 0))}
    if not name.startswith("k_topk"):
        path += (agg["dram_read"] + agg["dram_write"]) * n
    print(f"{name:32s} {n:2d} {agg['ms']:8.4f} {100 * agg['ms'] * n / tot_ms:5.1f}% {agg['dram_read'] / 1e9:10.3f} "
          f"{agg['dram_write'] / 1e9:10.3f} {agg.get('l2_hit_pct', 0):6.1f} {agg.get('issue_active_pct', 0):6.1f}")
try:
    with open(out_json) as fh:
        allj = json.load(fh)
except Exception:
    allj = {}
allj[config] = {"source": rep.split("/")[-1], "kernels": summary, "path_dram_bytes": int(path),
                "note": "ncu --set full --clock-control none, one counting path (cold, serialised replays)"}
with open(out_json, "w") as fh:
    json.dump(allj, fh, indent=1)
print("path DRAM bytes", int(path))
