#!/bin/bash
# A/B of settings at C2 on the GPU box (development aid): each argument is
# "label|ENV=V ENV2=V2|libpath" (empty env / lib: defaults); prints solve / V-cycle times
# and the per-level V-cycle costs for Jacobi and SOR, and checks the solutions bit for bit
# against the first variant.
mkdir -p gpurun_out/abv
out=gpurun_out/abv/summary.txt
: > $out
i=0
for spec in "$@"; do
  IFS='|' read -r label envs lib <<< "$spec"
  i=$((i+1))
  [ -n "$lib" ] && envs="$envs PF_LIB_PATH=$lib"
  echo "== $label ($envs)" >> $out
  env $envs timeout 300 python tools/ab_c2.py /tmp/abv_$i.npy >> $out 2>&1
  env $envs timeout 300 python tools/level_costs.py 7 0 2 >> $out 2>&1
  python -c "import numpy as np; a=np.load('/tmp/abv_1.npy'); b=np.load('/tmp/abv_$i.npy'); print('bit-identical to the first:', bool((a==b).all()))" >> $out 2>&1
done
