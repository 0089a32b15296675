#!/bin/bash
# compute-sanitizer over the kernel parity tests (SURVEY.md §5 race / memory evidence):
# memcheck (out-of-bounds / misaligned / leaks on the device), racecheck (shared-memory hazards),
# synccheck (barrier misuse), initcheck (reads of uninitialised device memory). Small scenes only
# (the tools slow kernels by 10-100x). Logs: gpurun_out/sanitize_<tool>.txt
set -x
mkdir -p gpurun_out
T_ALL=(tests/test_cull_gpu.py tests/test_raster_gpu.py tests/test_densify_gpu.py tests/test_split_engine_gpu.py tests/test_adam_gpu.py -k "not deferred_schedule_bitwise")
E=(tests/test_engine_gpu.py -k "serial_equals or delays or host_offload or step_async")
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  T=("${T_ALL[@]}")
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  # racecheck instruments every shared-memory access (100x+): the raster, cull and split tests only
  [ $tool = racecheck ] && T=(tests/test_cull_gpu.py tests/test_raster_gpu.py tests/test_split_engine_gpu.py -k "not reference")
  timeout ${SAN_T:-600} compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest "${T[@]}" -q -x -m gpu -p no:cacheprovider > gpurun_out/sanitize_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.txt
  timeout ${SAN_T:-600} compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest "${E[@]}" -q -x -m gpu -p no:cacheprovider > gpurun_out/sanitize_${tool}_engine.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_engine.txt
  tail -3 gpurun_out/sanitize_$tool.txt gpurun_out/sanitize_${tool}_engine.txt
done
