# vectorised gradient-unit loads in the deferred walk and the forwarding gather: A/B + parity
set -x
mkdir -p gpurun_out
for v in default gscalar default gscalar; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  GSS_LIB=$L timeout 300 python tools/adam_probe.py 40000000 0.1292 >> gpurun_out/adam_probe_ag.txt 2>&1
done
grep "{" gpurun_out/adam_probe_ag.txt
timeout 900 python -m pytest tests/test_adam_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/pytest_ag.txt 2>&1; tail -n 2 gpurun_out/pytest_ag.txt
