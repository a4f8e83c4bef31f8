# ncu --set full of one finest-level colour-sweep launch at C2: the TMA-staged kernel and
# the register-pipelined one (development aid); summaries under gpurun_out/.
set -x
mkdir -p gpurun_out/ncu
for v in tma off; do
  if [ $v = off ]; then export PF_SOR_TMA=0; K='k_color_sweep'; else unset PF_SOR_TMA; K='k_color_sweep_tma'; fi
  ncu --set full --clock-control none --import-source on -k "regex:^${K}\$" -s 12 -c 1 \
      -o /tmp/sor_$v -f python tools/profile_sweep.py 7 2 > gpurun_out/ncu/sor_$v.log 2>&1
  ncu -i /tmp/sor_$v.ncu-rep --page details --csv > gpurun_out/ncu/sor_${v}_details.csv
  ncu -i /tmp/sor_$v.ncu-rep --page raw --csv > gpurun_out/ncu/sor_${v}_raw.csv
  ncu -i /tmp/sor_$v.ncu-rep --page source --csv > gpurun_out/ncu/sor_${v}_source.csv 2>/dev/null
done
