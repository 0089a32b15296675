# staged (LDGSTS pipeline) deferred walk + forwarding gather: parity + isolated and in-step A/B vs the register walks
set -x
mkdir -p gpurun_out
B=paper_2509_15645_b200/_build
timeout 1500 python -m pytest tests/test_adam_gpu.py tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_densify_gpu.py "tests/test_scale_parity_gpu.py::test_c2_engine_three_iterations_vs_reference" -x -q > gpurun_out/pytest_au.txt 2>&1; tail -n 3 gpurun_out/pytest_au.txt
for i in 1 2; do
  for v in default wsprev ws4 ws2 ws3m3; do
    if [ $v = default ]; then L=; else L=$B/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 600 python tools/adam_probe.py > gpurun_out/ap_au_$v$i.json 2> gpurun_out/ap_au_$v.err
    python -c "import json;d=json.loads(open('gpurun_out/ap_au_$v$i.json').read());print('$v',{k:round(x,3) for k,x in d.items() if k.endswith(('ms','frac'))})" >> gpurun_out/ap_au.txt
  done
done
cat gpurun_out/ap_au.txt
for i in 1 2; do
  for v in default wsprev; do
    if [ $v = default ]; then L=; else L=$B/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_au_$v$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_au_$v$i.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),{k:round(v,3) for k,v in d['stage_ms_per_step'].items()},{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_au.txt
  done
done
cat gpurun_out/ab_au.txt
