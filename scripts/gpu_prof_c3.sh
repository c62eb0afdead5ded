#!/bin/bash
# ncu --set full of the C3 kernels: the apply (2nd launch), the sweep kernel, the volume kernel.
TAG=${1:-r02}
CFG=${2:-C3}
ncu --set full --clock-control none --import-source on -k "regex:k_apply|k_cg|k_volume|k_bicgstab" -s 2 -c 4 \
    -o gpurun_out/${TAG}_prof_${CFG} python scripts/prof_step.py ${CFG} > gpurun_out/${TAG}_prof_${CFG}.log 2>&1
tail -3 gpurun_out/${TAG}_prof_${CFG}.log
