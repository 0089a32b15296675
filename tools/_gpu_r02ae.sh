# cull grid in whole waves: bit-exactness (incl. 40M / 100M rows vs the oracle) and the kernel probe
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_cull_gpu.py "tests/test_scale_parity_gpu.py::test_cull_beyond_co_residency_vs_oracle" -x -q > gpurun_out/pytest_ae.txt 2>&1; tail -n 2 gpurun_out/pytest_ae.txt
timeout 1200 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-host-offload > gpurun_out/bench_ae.json 2> gpurun_out/bench_ae.err
python -c "import json;d=json.loads(open('gpurun_out/bench_ae.json').read().strip().splitlines()[-1]);print(d['value'],d['stage_ms_per_step']['cull'],[(k['kernel'][:14],round(k['ms'],4),round(k['frac'],3)) for k in d['kernels']])"
