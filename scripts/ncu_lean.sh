#!/bin/bash
# one lean-kernel interior solve under ncu (kernel replay): source-level stall samples
N=${1:-256}
ncu --set full --import-source on --clock-control none -k regex:sptrsv_lean --launch-skip 3 --launch-count 1 \
    -f -o gpurun_out/r1c_lean_ncu python scripts/probe_tiled.py --n $N --kernel warp --no-sell --out gpurun_out/ncu_probe.jsonl > gpurun_out/ncu_lean.log 2>&1
tail -3 gpurun_out/ncu_lean.log
