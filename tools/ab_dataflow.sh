# A/B of the dataflow colour sweep against the per-colour launches: C2 (8-bit values),
# 64^3, lognormal C2 (fp64); solutions compared bit for bit.  TILTS: PF_SOR_DF_TILT values
# ("" = the default formula).
mkdir -p gpurun_out/df /tmp/df
for L in 7 6; do
  PF_SOR_DATAFLOW=0 python tools/ab_c2.py /tmp/df/s_off_$L.npy $L > gpurun_out/df/c_off_$L.txt 2>&1
  echo "== dataflow off L=$L" >> gpurun_out/df/summary.txt; grep "kind 2" gpurun_out/df/c_off_$L.txt >> gpurun_out/df/summary.txt
  for t in ${TILTS:-default 100000000}; do
    if [ $t = default ]; then unset PF_SOR_DF_TILT; else export PF_SOR_DF_TILT=$t; fi
    python tools/ab_c2.py /tmp/df/s_$L.npy $L > gpurun_out/df/c_${t}_$L.txt 2>&1
    python -c "
import numpy as np
print('== dataflow tilt=$t L=$L identical:', np.array_equal(np.load('/tmp/df/s_off_$L.npy'), np.load('/tmp/df/s_$L.npy')))" >> gpurun_out/df/summary.txt
    grep "kind 2" gpurun_out/df/c_${t}_$L.txt >> gpurun_out/df/summary.txt
  done
  unset PF_SOR_DF_TILT
done
for v in 0 1; do echo "== lognormal dataflow=$v" >> gpurun_out/df/summary.txt; PF_SOR_DATAFLOW=$v python tools/lognormal_c2.py 2>&1 | grep "kind 2\|SOR" >> gpurun_out/df/summary.txt; done
