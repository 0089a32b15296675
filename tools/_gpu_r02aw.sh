# handoff(g) on a side stream beside geo_update(g) (stream D waits for it before cull(g+1)): engine parity + same-box A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_densify_gpu.py tests/test_dropin_gpu.py "tests/test_scale_parity_gpu.py::test_c2_engine_three_iterations_vs_reference" -x -q > gpurun_out/pytest_aw.txt 2>&1; tail -n 3 gpurun_out/pytest_aw.txt
for i in 1 2 3; do
  for v in 1 0; do
    GSS_HANDOFF_SIDE=$v timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_aw_$v$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_aw_$v$i.json').read().strip().splitlines()[-1]);print('side=$v',round(d['value'],3),round(d['e2e']['value'],3),{k:round(v,3) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/ab_aw.txt
  done
done
cat gpurun_out/ab_aw.txt
