# ncu --set full of one finest-level k_jacobi launch at 384^3 with the identity and the
# colour-interleaved block schedule.
mkdir -p gpurun_out/ncu
for v in 100000000000 67108864; do
  PF_INTERLEAVE_MIN_BYTES=$v ncu --set full --clock-control none -k "regex:^k_jacobi\$" -s 5 -c 1 \
      -o /tmp/large_$v -f python tools/profile_large_sweep.py 3 8 0 > gpurun_out/ncu/large_$v.log 2>&1
  ncu -i /tmp/large_$v.ncu-rep --page details --csv > gpurun_out/ncu/large_${v}_details.csv
  ncu -i /tmp/large_$v.ncu-rep --page raw --csv > gpurun_out/ncu/large_${v}_raw.csv
done
