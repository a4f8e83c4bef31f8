# A/B of the colour sweep variants at C2 (8-bit values) and lognormal C2 (fp64 values).
mkdir -p gpurun_out/ab2 /tmp/ab
PF_SOR_WIDE=0 python tools/ab_c2.py /tmp/ab/base.npy 7 > gpurun_out/ab2/base.txt 2>&1
PF_SOR_WIDE=1 python tools/ab_c2.py /tmp/ab/wide.npy 7 > gpurun_out/ab2/wide.txt 2>&1
python -c "
import numpy as np
print('identical:', np.array_equal(np.load('/tmp/ab/base.npy'), np.load('/tmp/ab/wide.npy')))" > gpurun_out/ab2/summary.txt
for f in base wide; do echo "== $f" >> gpurun_out/ab2/summary.txt; grep "kind 2" gpurun_out/ab2/$f.txt >> gpurun_out/ab2/summary.txt; done
for f in 0 1; do echo "== lognormal wide=$f" >> gpurun_out/ab2/summary.txt; PF_SOR_WIDE=$f python tools/lognormal_c2.py 2>&1 | grep "kind 2\|SOR" >> gpurun_out/ab2/summary.txt; done
