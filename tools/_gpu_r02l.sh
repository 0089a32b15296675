# full gpu suite, C4 launch list of a short bench, sanitizer logs
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_l.txt 2>&1
tail -3 gpurun_out/pytest_l.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench.log 2>&1
tail -2 gpurun_out/launch_bench.log
SAN_T=500 bash tools/sanitize.sh > gpurun_out/sanitize_driver.txt 2>&1
tail -20 gpurun_out/sanitize_driver.txt
