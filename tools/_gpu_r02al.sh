# composite occupancy A/B (CTAs per SM via register caps) from the bench's composite ms
set -x
mkdir -p gpurun_out
for v in default fmb9 fmb10 default; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_al_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench_al_$v.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_al.txt
done
cat gpurun_out/ab_al.txt
