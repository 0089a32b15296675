# row-staged (TMA bulk) deferred walk + forwarding gather: parity + isolated A/B vs the register walks
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_adam_gpu.py tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_densify_gpu.py -x -q > gpurun_out/pytest_ar.txt 2>&1; tail -n 3 gpurun_out/pytest_ar.txt
for i in 1 2; do
  for v in default wbprev wbs2m3 wbs4 wbr16; do
    if [ $v = default ]; then L=; else L=paper_2509_15645_b200/_build/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 600 python tools/adam_probe.py >> gpurun_out/adam_probe_ar.jsonl 2> gpurun_out/adam_probe_ar_$v.err
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/adam_probe_ar.jsonl'):
    d=json.loads(l); print(d['lib'].split('/')[-2] if '/' in d['lib'] else d['lib'], {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.items() if k not in ('lib','n','frac')})
PY
for i in 1 2; do
  for v in default wbprev; do
    if [ $v = default ]; then L=; else L=paper_2509_15645_b200/_build/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_ar_$v$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_ar_$v$i.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),{k:round(v,3) for k,v in d['stage_ms_per_step'].items()},{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_ar.txt
  done
done
cat gpurun_out/ab_ar.txt
