# final round-2 evidence after the folded exp factor: full GPU suite, smoke, default bench, launch list
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_bb.txt 2>&1; tail -n 3 gpurun_out/pytest_bb.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_bb.txt 2>&1; tail -n 1 gpurun_out/smoke_bb.txt
( time timeout 1200 python bench.py > gpurun_out/bench_c4_bb.json 2> gpurun_out/bench_c4_bb.err ) 2> gpurun_out/bench_c4_bb.time
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_bb.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['render_kernels']['phases_ms_per_step'],[(k['kernel'][:12],round(k['frac'],3)) for k in d['kernels']],d['host_offload']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_bb.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench_bb.log 2>&1
