# compute-sanitizer evidence (memcheck / racecheck / synccheck / initcheck) over the kernel and engine tests
set -x
mkdir -p gpurun_out
SAN_T=420 bash tools/sanitize.sh > gpurun_out/sanitize_driver.txt 2>&1
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|LEAK SUMMARY\|passed\|failed\|^exit" gpurun_out/sanitize_*.txt | head -40
