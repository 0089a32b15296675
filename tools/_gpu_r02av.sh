# evidence on the head with the leaner sweep (dx-factored moments, one select per idle pixel)
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_av.txt 2>&1; tail -n 3 gpurun_out/pytest_av.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_av.txt 2>&1; tail -n 1 gpurun_out/smoke_av.txt
( time timeout 1200 python bench.py > gpurun_out/bench_c4_av.json 2> gpurun_out/bench_c4_av.err ) 2> gpurun_out/bench_c4_av.time
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_av.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['render_kernels']['phases_ms_per_step'],[(k['kernel'][:12],round(k['frac'],3)) for k in d['kernels']],d['host_offload']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_av.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench_av.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:backward_kernel -c 1 -o gpurun_out/c4_bwd_av python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_bwd_av.txt 2>&1
tail -n 1 gpurun_out/ncu_bwd_av.txt
