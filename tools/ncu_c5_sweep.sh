# ncu --set full of finest-level k_color_sweep launches (multicolour SOR, fp64 values: the
# lognormal coefficient) at 384^3 — the kernel and operator kind of the C5 scaling
# configuration at a size whose setup takes under a minute.  Outputs in gpurun_out/ncu/.
mkdir -p gpurun_out/ncu
python tools/profile_large_sweep.py 3 8 2 4 > gpurun_out/ncu/c5_sweep_plain.log 2>&1 &&
ncu --set full --clock-control none -k "regex:^k_color_sweep" -s 26 -c 2 \
    -o /tmp/c5_sweep -f python tools/profile_large_sweep.py 3 8 2 4 > gpurun_out/ncu/c5_sweep.log 2>&1
ncu -i /tmp/c5_sweep.ncu-rep --page details --csv > gpurun_out/ncu/c5_sweep_details.csv
ncu -i /tmp/c5_sweep.ncu-rep --page raw --csv > gpurun_out/ncu/c5_sweep_raw.csv
tail -2 gpurun_out/ncu/c5_sweep_plain.log
