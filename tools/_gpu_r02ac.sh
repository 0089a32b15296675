# round-end candidate: full GPU suite, memcheck + initcheck over the raster/engine tests with the final kernels, full bench
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ac.txt 2>&1; tail -n 3 gpurun_out/pytest_ac.txt
for tool in memcheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_raster_gpu.py tests/test_split_engine_gpu.py tests/test_imgpar_gpu.py -q -x -m gpu -p no:cacheprovider -k "not two_process" > gpurun_out/sanitize2_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize2_$tool.txt
  grep "ERROR SUMMARY\|passed\|failed\|^exit" gpurun_out/sanitize2_$tool.txt
done
( time timeout 1200 python bench.py > gpurun_out/bench_c4_ac.json 2> gpurun_out/bench_c4_ac.err ) 2> gpurun_out/bench_c4_ac.time
tail -c 200 gpurun_out/bench_c4_ac.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ac.txt 2>&1; tail -n 2 gpurun_out/smoke_ac.txt
