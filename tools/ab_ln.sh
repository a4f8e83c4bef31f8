#!/bin/bash
# lognormal C2 A/B (development aid): tools/ab_ln.sh "ENV.." "ENV.." ...
for rep in 1 2; do
  i=0
  for a in "$@"; do
    i=$((i+1))
    echo "== [$i] $a (run $rep)" >> gpurun_out/ab_ln.log
    env $a timeout 300 python tools/lognormal_c2.py 2>&1 | grep -v "^{" >> gpurun_out/ab_ln.log
  done
done
