# Round profiling pass (one GPU): the C2 Jacobi solve's launch list (host-driven outer loop,
# so ncu sees the graph's kernel nodes) and one ncu --set full capture of the finest
# k_jacobi; outputs in gpurun_out/prof/.
mkdir -p gpurun_out/prof
PF_SOLVE_MODE=host ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_c2_jacobi.csv python tools/one_solve.py 7 0 > gpurun_out/prof/launches.log 2>&1
PF_SOLVE_MODE=host ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_c2_sor.csv python tools/one_solve.py 7 2 > gpurun_out/prof/launches_sor.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_jacobi\$" -s 3 -c 1 \
    -o /tmp/k_jacobi_c2 -f python tools/profile_sweep.py 7 0 > gpurun_out/prof/k_jacobi.log 2>&1
ncu -i /tmp/k_jacobi_c2.ncu-rep --page raw --csv > gpurun_out/prof/k_jacobi_c2_raw.csv
ncu -i /tmp/k_jacobi_c2.ncu-rep --page details --csv > gpurun_out/prof/k_jacobi_c2_details.csv
