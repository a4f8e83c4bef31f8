# SOR sweep at a large grid (x >> L2) with the per-colour launches and the dataflow kernel.
mkdir -p gpurun_out/lsor
for v in "PF_SOR_DATAFLOW=0" "PF_SOR_DATAFLOW=1"; do
  env $v python tools/profile_large_sweep.py ${NC:-3} ${LV:-8} 2 ${PROB:-4} > gpurun_out/lsor/one.txt 2>&1
  echo "== $v" >> gpurun_out/lsor/summary.txt; cat gpurun_out/lsor/one.txt >> gpurun_out/lsor/summary.txt
done
