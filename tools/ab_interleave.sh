mkdir -p gpurun_out/il
for v in ${VARIANTS:-"PF_INTERLEAVE_MIN_BYTES=100000000000" "PF_INTERLEAVE_AHEAD=0" "PF_INTERLEAVE_AHEAD=48" "PF_INTERLEAVE_AHEAD=96" "PF_INTERLEAVE_AHEAD=192"}; do
  env $v python tools/ab_interleave.py ${NC:-3} ${LV:-8} ${PROB:-0} > gpurun_out/il/one.txt 2>&1
  echo "== $v" >> gpurun_out/il/summary.txt; cat gpurun_out/il/one.txt >> gpurun_out/il/summary.txt
done
