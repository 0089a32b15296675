# debug: in-place host-tier arena passes under compute-sanitizer; forward clamp-free timing
set -x
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest -x -q "tests/test_adam_gpu.py::test_host_tier_arena_passes_bitwise" > gpurun_out/san_k.txt 2>&1
grep -m 30 -E "Invalid|at 0x|by thread|Address|kernel|passed|failed" gpurun_out/san_k.txt | head -30
timeout 300 python tools/time_render.py 40000000 3840 2160 > gpurun_out/time_render_c4_k.txt 2>&1
tail -9 gpurun_out/time_render_c4_k.txt
