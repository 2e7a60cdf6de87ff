#!/bin/bash
# Launch list (gpu__time_duration, cold-cache serialised) of one search of a workload.
#   tools/ncu_launches.sh OUT.csv [config] [flat partition cells]
out=${1:-gpurun_out/launches.csv}
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out" \
    python tools/profile_step.py ${2:-config1} ${3:-} > /dev/null 2>&1
