# correctness of the new forward, A/B timing, then the default bench (C4 headline) + reference arm
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --ignore=tests/test_scale_parity_gpu.py > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python tools/time_render.py 40000000 3840 2160 2 > gpurun_out/time_c4_new.txt 2>&1
GSS_LIB=paper_2509_15645_b200/_build/var_coefldc/libgss_b200.so timeout 600 python tools/time_render.py 40000000 3840 2160 2 > gpurun_out/time_c4_coefldc.txt 2>&1
tail -1 gpurun_out/time_c4_new.txt gpurun_out/time_c4_coefldc.txt
( time timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err ) 2> gpurun_out/bench_c4.time
( time timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err ) 2> gpurun_out/bench_ref.time
tail -c 600 gpurun_out/bench_c4.err; tail -c 600 gpurun_out/bench_ref.err; cat gpurun_out/*.time
