#!/bin/bash
# A/B of library builds at C2 on the GPU box (development aid):
#   tools/ab_lib.sh build_variants/x/libpf_gpu.so [...]   (the in-tree library is the baseline)
timeout 300 python tools/ab_c2.py /tmp/base.npy > gpurun_out/ab_base.log 2>&1
i=0
for lib in "$@"; do
  i=$((i+1))
  PF_LIB_PATH=$lib timeout 300 python tools/ab_c2.py /tmp/v$i.npy > gpurun_out/ab_v$i.log 2>&1
  python -c "import numpy as np; a=np.load('/tmp/base.npy'); b=np.load('/tmp/v$i.npy'); print('$lib bitexact', [bool((a[k]==b[k]).all()) for k in range(len(a))])" >> gpurun_out/ab_v$i.log 2>&1
done
timeout 300 python tools/ab_c2.py /tmp/base2.npy > gpurun_out/ab_base2.log 2>&1
