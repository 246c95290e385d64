#!/bin/bash
# ncu --set full of the full-block pass of the blocked Gram-Schmidt (256^3 outer basis)
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:mgs_block_kernel<.int.4, .int.4>' -s 20 -c 3 -f -o gpurun_out/r1c_prof_mgs44 \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_mgs44.log 2>&1
tail -2 gpurun_out/ncu_mgs44.log | cut -c1-200
