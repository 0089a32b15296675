# default bench (C4 headline) + reference arm, timed by the wall clock
set -x
mkdir -p gpurun_out
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
/usr/bin/time -v timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 600 gpurun_out/bench_c4.err; tail -c 600 gpurun_out/bench_ref.err
