#!/bin/bash
# One GPU call: the default bench line, its ncu launch list (same workload, no extras / CPU
# baseline), and one full ncu capture of the dominant kernel. Outputs in gpurun_out/$TAG*.
TAG=${1:-r02}
KREGEX=${2:-regex:k_cg_w}
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 3000 gpurun_out/${TAG}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline \
    > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k "$KREGEX" -s 2 -c 1 \
    -o gpurun_out/${TAG}_top python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline \
    > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out/
