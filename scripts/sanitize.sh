# compute-sanitizer over every kernel at smoke size (scripts/sanitize_driver.py); logs to gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, extra flags, driver parts
  tool=$1; shift; extra=$1; shift
  timeout 1200 $CS --tool $tool $extra --error-exitcode 9 python scripts/sanitize_driver.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  grep -E "ERROR SUMMARY|LEAK SUMMARY|RACECHECK SUMMARY|rc=" gpurun_out/sanitize_$tool.log | tail -3
}
run memcheck "--leak-check full"
# the resident service kernel polls mapped host memory for its whole life: memcheck only
run racecheck "--racecheck-report all" sim seg simtput bulk tk metrics wl single
run synccheck "" sim seg simtput bulk tk metrics wl single
run initcheck "" sim seg simtput bulk tk metrics wl single
