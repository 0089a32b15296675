# certified-range composite as default: adversarial + full raster parity (both variants), racecheck on the
# cull ring with the refill fences, full bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_raster_gpu.py tests/test_cull_gpu.py -x -q > gpurun_out/pytest_v.txt 2>&1; tail -2 gpurun_out/pytest_v.txt
GSS_LIB=paper_2509_15645_b200/_build/var_fchecked/libgss_b200.so timeout 900 python -m pytest tests/test_raster_gpu.py -x -q -k adversarial > gpurun_out/pytest_v_checked.txt 2>&1; tail -2 gpurun_out/pytest_v_checked.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_cull_gpu.py -q -x -m gpu -p no:cacheprovider -k "acceptance or random" > gpurun_out/sanitize_racecheck_cull.txt 2>&1; echo "exit $?" >> gpurun_out/sanitize_racecheck_cull.txt
grep "RACECHECK SUMMARY\|passed\|exit\|hazard" gpurun_out/sanitize_racecheck_cull.txt | sort | uniq -c | head
( time timeout 1200 python bench.py > gpurun_out/bench_c4_v.json 2> gpurun_out/bench_c4_v.err ) 2> gpurun_out/bench_c4_v.time
tail -c 200 gpurun_out/bench_c4_v.err
