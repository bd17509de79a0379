#!/bin/bash
# ncu captures of the c2 counting path (run on the GPU box from the repo root):
#   1. launch list of the bench command (per-launch times, cold and serialised)
#   2. one `--set full` capture of every kernel of the third pass of the path
# Summaries: python tools/launches.py gpurun_out/launches_c2.csv,
#            python tools/ncu_summary.py gpurun_out/c2_path.ncu-rep c2
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(item_terms|plan_stream|chunk_bounds|scan_u64|stream_scatter|stream_count|stream_write|count_stream|reduce_slabs|topk)" \
    --launch-skip 20 --launch-count 10 -o gpurun_out/c2_path -f \
    python tools/quick_pairs.py c2 > gpurun_out/ncu_full.log 2>&1
