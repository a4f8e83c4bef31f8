#!/bin/bash
# tools/ab_lib.sh plus the L=6 (64^3) hierarchy (development aid)
tools/ab_lib.sh "$@"
for L in 6; do
  timeout 200 python tools/ab_c2.py /tmp/x.npy $L | grep kind > gpurun_out/abL_base.log 2>&1
  i=0
  for lib in "$@"; do i=$((i+1)); PF_LIB_PATH=$lib timeout 200 python tools/ab_c2.py /tmp/x.npy $L | grep kind > gpurun_out/abL_v$i.log 2>&1; done
done
