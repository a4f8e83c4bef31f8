# A/B of the colour sweep kernels at C2 (and 64^3): register-pipelined vs TMA-staged
# (PF_SOR_TMA_CFG configurations x blocks per SM); solutions compared bit for bit.
mkdir -p gpurun_out/ab /tmp/ab
for L in ${LEVELS:-7}; do
PF_SOR_TMA=0 python tools/ab_c2.py /tmp/ab/off_$L.npy $L > gpurun_out/ab/off_$L.txt 2>&1
echo "== off L=$L" >> gpurun_out/ab/summary.txt; grep "kind 2" gpurun_out/ab/off_$L.txt >> gpurun_out/ab/summary.txt
for cfg in ${CFG_LIST:-0 1 2}; do
for bps in ${BPS_LIST:-1 2 3}; do
PF_SOR_TMA_CFG=$cfg PF_SOR_TMA_BPS=$bps python tools/ab_c2.py /tmp/ab/t_$L.npy $L > gpurun_out/ab/t_${cfg}_${bps}_$L.txt 2>&1
python -c "
import numpy as np
a=np.load('/tmp/ab/off_$L.npy'); b=np.load('/tmp/ab/t_$L.npy')
print('== tma cfg=$cfg bps=$bps L=$L identical:', np.array_equal(a,b))" >> gpurun_out/ab/summary.txt
grep "kind 2" gpurun_out/ab/t_${cfg}_${bps}_$L.txt >> gpurun_out/ab/summary.txt
done; done; done
