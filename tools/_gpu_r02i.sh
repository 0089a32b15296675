# ncu source-level capture of the composite and sweep at C4 (one launch each, camera 1)
set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"forward_kernel|backward_kernel" -s 2 -c 2 -o gpurun_out/c4_raster_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_src.txt 2>&1
tail -3 gpurun_out/ncu_src.txt
ls -la gpurun_out/
