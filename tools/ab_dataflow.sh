# A/B of the dataflow colour sweep against the per-colour launches: C2 (8-bit values),
# 64^3, lognormal C2 (fp64); solutions compared bit for bit.
mkdir -p gpurun_out/df /tmp/df
for L in 7 6; do
  for v in 0 1; do PF_SOR_DATAFLOW=$v python tools/ab_c2.py /tmp/df/s_${v}_$L.npy $L > gpurun_out/df/c_${v}_$L.txt 2>&1; done
  python -c "
import numpy as np
print('L=$L identical:', np.array_equal(np.load('/tmp/df/s_0_$L.npy'), np.load('/tmp/df/s_1_$L.npy')))" >> gpurun_out/df/summary.txt
  for v in 0 1; do echo "== dataflow=$v L=$L" >> gpurun_out/df/summary.txt; grep "kind 2" gpurun_out/df/c_${v}_$L.txt >> gpurun_out/df/summary.txt; done
done
for v in 0 1; do echo "== lognormal dataflow=$v" >> gpurun_out/df/summary.txt; PF_SOR_DATAFLOW=$v python tools/lognormal_c2.py 2>&1 | grep "kind 2\|SOR" >> gpurun_out/df/summary.txt; done
