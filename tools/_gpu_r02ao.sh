# concurrent host tier (lazy(g-1) beside fp(g) on disjoint rows): parity + A/B at C3 / C4
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_densify_gpu.py tests/test_adam_gpu.py "tests/test_scale_parity_gpu.py::test_c3_offload_two_iterations_vs_reference" -x -q > gpurun_out/pytest_ao.txt 2>&1; tail -n 2 gpurun_out/pytest_ao.txt
run() {  # tag, n, w, h, env...
  tag=$1; n=$2; w=$3; h=$4; shift 4
  env "$@" timeout 900 python bench.py --n $n --width $w --height $h --nongeo-tier host --no-cpu-baseline --no-probe --no-host-offload --steps 8 --warmup 8 > gpurun_out/hostc_$tag.json 2> gpurun_out/hostc_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/hostc_$tag.json').read().strip().splitlines()[-1]);print('$tag',round(d['value'],3),{k:round(v,1) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/hostc_ab.txt
}
run c3_serialorder 18000000 1920 1080 GSS_HOST_CONCURRENT=0
run c3_concurrent 18000000 1920 1080 X=1
run c4_serialorder 40000000 3840 2160 GSS_HOST_CONCURRENT=0
run c4_concurrent 40000000 3840 2160 X=1
cat gpurun_out/hostc_ab.txt
