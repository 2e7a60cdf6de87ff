#!/bin/bash
# Launch list (gpu__time_duration) of this repo's kernels during one phase_profile run.
#   tools/ncu_launches.sh OUT.csv [config]
out=${1:-gpurun_out/launches.csv}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out" \
    -k regex:"rotate|sq_norms|coarse|group_|fill_u32|row_norms|seed_|dco_|advance_surv|scan_counts|scatter_cand|merge_|tighten|keys_to" \
    python tools/phase_profile.py ${2:-config1} > /dev/null 2>&1
