#!/bin/bash
# ncu --set full of one finest-level sweep kernel at C2 (development aid).
#   tools/ncu_sweep.sh <kernel-regex> <out-name> [levels] [kind]
set -e
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:^$1\$" -s 3 -c 1 \
    -o gpurun_out/$2 -f python tools/profile_sweep.py ${3:-7} ${4:-0} > gpurun_out/$2.log 2>&1
ncu -i gpurun_out/$2.ncu-rep --page raw --csv > gpurun_out/$2_raw.csv
ncu -i gpurun_out/$2.ncu-rep --page details --csv > gpurun_out/$2_details.csv
ncu -i gpurun_out/$2.ncu-rep --page source --csv > gpurun_out/$2_source.csv || true
