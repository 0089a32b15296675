# stream priority A/B at C4 (render phases per step)
set -x
mkdir -p gpurun_out
for m in 0 1 2 0; do
  GSS_STREAM_PRIO=$m timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_ab_p$m.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench_ab_p$m.json').read().strip().splitlines()[-1]);print('prio $m',round(d['value'],3),{k:round(v,2) for k,v in d['stage_ms_per_step'].items()},{k:round(v,2) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_prio.txt
done
cat gpurun_out/ab_prio.txt
