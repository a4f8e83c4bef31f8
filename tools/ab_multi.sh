#!/bin/bash
# A/B of several settings at C2 (development aid): tools/ab_multi.sh "ENV=.." "ENV=.. PF_LIB_PATH=.." ...
# (the first argument is the baseline; each setting runs twice, interleaved; solutions compared)
L=${AB_LEVELS:-7}
for rep in 1 2; do
  i=0
  for a in "$@"; do
    i=$((i+1))
    echo "== [$i] $a (run $rep)" >> gpurun_out/ab_multi.log
    env $a timeout 300 python tools/ab_c2.py /tmp/s$i.npy $L >> gpurun_out/ab_multi.log 2>&1
  done
done
i=0
for a in "$@"; do
  i=$((i+1))
  python -c "import numpy as np; a=np.load('/tmp/s1.npy'); b=np.load('/tmp/s$i.npy'); print('[$i] bitexact vs [1]', [bool((a[k]==b[k]).all()) for k in range(len(a))])" >> gpurun_out/ab_multi.log 2>&1
done
