#!/bin/bash
# A/B of an environment setting at C2 on the GPU box: tools/ab_run.sh "VAR=0" (development aid)
A="$1"
env $A timeout 300 python tools/ab_c2.py /tmp/a.npy > gpurun_out/ab_a.log 2>&1
timeout 300 python tools/ab_c2.py /tmp/b.npy > gpurun_out/ab_b.log 2>&1
env $A timeout 300 python tools/ab_c2.py /tmp/a2.npy > gpurun_out/ab_a2.log 2>&1
timeout 300 python tools/ab_c2.py /tmp/b2.npy > gpurun_out/ab_b2.log 2>&1
python -c "import numpy as np; a=np.load('/tmp/a.npy'); b=np.load('/tmp/b.npy'); print('bitexact', [bool((a[i]==b[i]).all()) for i in range(len(a))])" > gpurun_out/ab_cmp.log 2>&1
