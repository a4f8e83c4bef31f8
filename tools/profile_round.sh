# Round profiling pass (one GPU): the C2 Jacobi and SOR solves' launch lists (host-driven
# outer loop, so ncu sees the graph's kernel nodes), one ncu --set full capture of the
# finest k_jacobi (the bench's roofline kernel), and of the mid-level wide colour sweep and
# the one-block bottom kernel of the SOR cycle.  Each ncu command runs only after the same
# command exited 0 without ncu.  Outputs in gpurun_out/prof/.
mkdir -p gpurun_out/prof
P=gpurun_out/prof
PF_SOLVE_MODE=host python tools/one_solve.py 7 0 > $P/plain_j.log 2>&1 &&
PF_SOLVE_MODE=host ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $P/launches_c2_jacobi.csv python tools/one_solve.py 7 0 > $P/launches.log 2>&1
PF_SOLVE_MODE=host python tools/one_solve.py 7 2 > $P/plain_s.log 2>&1 &&
PF_SOLVE_MODE=host ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $P/launches_c2_sor.csv python tools/one_solve.py 7 2 > $P/launches_sor.log 2>&1
python tools/profile_sweep.py 7 0 > $P/plain_sweep.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:^k_jacobi\$" -s 3 -c 1 \
    -o /tmp/k_jacobi_c2 -f python tools/profile_sweep.py 7 0 > $P/k_jacobi.log 2>&1
ncu -i /tmp/k_jacobi_c2.ncu-rep --page raw --csv > $P/k_jacobi_c2_raw.csv
ncu -i /tmp/k_jacobi_c2.ncu-rep --page details --csv > $P/k_jacobi_c2_details.csv
python tools/vcycle_profile.py 2 > $P/plain_vc.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:k_color_sweep_wide|k_bottom_block" -c 2 \
    -o /tmp/sor_small -f python tools/vcycle_profile.py 2 > $P/sor_small.log 2>&1
ncu -i /tmp/sor_small.ncu-rep --page details --csv > $P/sor_small_details.csv
