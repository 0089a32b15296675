# host tier: render/zero-copy interference A/B (serialised render, host-pass grid size) at C3 and C4
set -x
mkdir -p gpurun_out
run() {  # tag, n, w, h, env...
  tag=$1; n=$2; w=$3; h=$4; shift 4
  env "$@" timeout 900 python bench.py --n $n --width $w --height $h --nongeo-tier host --no-cpu-baseline --no-probe --no-host-offload --steps 8 --warmup 8 > gpurun_out/host_$tag.json 2> gpurun_out/host_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/host_$tag.json').read().strip().splitlines()[-1]);print('$tag',round(d['value'],3),{k:round(v,1) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/host_ab.txt
}
run c3_base 18000000 1920 1080 X=0
run c3_serial 18000000 1920 1080 GSS_HOST_SERIAL=1
run c3_b16 18000000 1920 1080 GSS_HOST_BLOCKS=16
run c3_serial_b32 18000000 1920 1080 GSS_HOST_SERIAL=1 GSS_HOST_BLOCKS=32
run c4_base 40000000 3840 2160 X=0
run c4_serial 40000000 3840 2160 GSS_HOST_SERIAL=1
cat gpurun_out/host_ab.txt
