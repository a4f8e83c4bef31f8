# compute-sanitizer over every kernel family (tools/sanitize_run.py); logs to
# gpurun_out/sanitizer/.  Each run is bounded by timeout.
mkdir -p gpurun_out/sanitizer
CS="compute-sanitizer --error-exitcode 9 --print-limit 50"
run() {  # name tool env... -- phases
  local name=$1 tool=$2; shift 2
  local envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout ${TMO:-900} $CS --tool $tool python tools/sanitize_run.py "$@" > gpurun_out/sanitizer/${name}.log 2>&1
  echo "$name rc=$? $(grep -c 'phase .* ok' gpurun_out/sanitizer/${name}.log) phases ok; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer/${name}.log | tr '\n' ' ')" >> gpurun_out/sanitizer/summary.txt
}
run memcheck_default memcheck PF_X=1 --
run memcheck_host_loop memcheck PF_SOLVE_MODE=host --
run memcheck_variants memcheck PF_SOR_TMA=1 PF_SOR_TMA_MIN_ROWS=0 PF_INTERLEAVE_MIN_BYTES=0 -- jacobi_k1 sor_k2 gs_k4_lognormal fe
run racecheck_default racecheck PF_X=1 -- jacobi_k1 sor_k2 gs_k4_lognormal loopback_k2 heat
run racecheck_tma racecheck PF_SOR_TMA=1 PF_SOR_TMA_MIN_ROWS=0 -- sor_k2 fe
run synccheck_default synccheck PF_X=1 --
run initcheck_default initcheck PF_X=1 -- jacobi_k1 sor_k2 loopback_k2 heat
cat gpurun_out/sanitizer/summary.txt
