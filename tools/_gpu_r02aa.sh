# full bench at C4 with render phase breakdown; C3 host-tier bench with the tuned host grids
set -x
mkdir -p gpurun_out
( time timeout 1200 python bench.py > gpurun_out/bench_c4_aa.json 2> gpurun_out/bench_c4_aa.err ) 2> gpurun_out/bench_c4_aa.time
tail -c 200 gpurun_out/bench_c4_aa.err
timeout 900 python bench.py --n 18000000 --width 1920 --height 1080 --nongeo-tier host --no-cpu-baseline --no-probe --no-host-offload --steps 8 --warmup 8 > gpurun_out/bench_c3_host_aa.json 2> gpurun_out/bench_c3_host_aa.err
tail -c 200 gpurun_out/bench_c3_host_aa.err
