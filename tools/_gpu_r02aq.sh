# evidence refresh on the re-entry head (after the certified-composite and concurrent host-tier commits)
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_aq.txt 2>&1; tail -n 3 gpurun_out/pytest_aq.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_aq.txt 2>&1; tail -n 1 gpurun_out/smoke_aq.txt
( time timeout 1200 python bench.py > gpurun_out/bench_c4_aq.json 2> gpurun_out/bench_c4_aq.err ) 2> gpurun_out/bench_c4_aq.time
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_aq.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['render_kernels']['phases_ms_per_step'],[(k['kernel'][:12],round(k['frac'],3)) for k in d['kernels']],d['host_offload']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_aq.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench_aq.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:backward_kernel -c 1 -o gpurun_out/c4_bwd_aq python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_bwd_aq.txt 2>&1
tail -n 1 gpurun_out/ncu_bwd_aq.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:forward_kernel -c 1 -o gpurun_out/c4_fwd_aq python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_fwd_aq.txt 2>&1
tail -n 1 gpurun_out/ncu_fwd_aq.txt
