# host-tier pass grid sizes (isolated passes at C3 scale), then the C3 host-tier bench at the best pair
set -x
mkdir -p gpurun_out
for rb in 8 16 32 64; do
  for wb in 16 32 64 128 256; do
    echo -n "rb=$rb wb=$wb " >> gpurun_out/host_grid.txt
    GSS_HOST_BLOCKS=$rb GSS_HOST_WALK_BLOCKS=$wb timeout 300 python tools/host_tier_probe.py 18000000 0.145 2>/dev/null | tail -n 1 >> gpurun_out/host_grid.txt
  done
done
cat gpurun_out/host_grid.txt
