# The in-process peer transport (tests/peer_threads.py) over a few shapes; PF_TRACE=1 shows
# where each rank is.
mkdir -p gpurun_out/exp1
for args in "--world 8 --levels 3 --rep coarse" "--world 8 --levels 4 --rep bottom --fused" "--world 4 --levels 4 --rep bottom --fused --kind 2" "--world 2 --levels 4 --rep coarse"; do
  d=$(mktemp -d); t0=$(date +%s)
  CUDA_MODULE_LOADING=EAGER CUDA_DEVICE_MAX_CONNECTIONS=32 PF_WATCHDOG_S=${WD:-10} timeout 200 python tests/peer_threads.py --out $d $args > gpurun_out/exp1/out.txt 2>&1; rc=$?
  echo "[$args] rc=$rc $(( $(date +%s) - t0 )) s $(ls $d | wc -l) files $(tail -c 300 gpurun_out/exp1/out.txt)" >> gpurun_out/exp1/log.txt
done
