# C4 strip parity vs the reference renderer; launch list; ncu of the final composite + sweep
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest "tests/test_scale_parity_gpu.py::test_c4_strip_forward_backward_vs_reference" -x -q > gpurun_out/pytest_w.txt 2>&1; tail -n 3 gpurun_out/pytest_w.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_w.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench_w.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:forward_kernel -s 8 -c 1 -o gpurun_out/c4_fwd_final python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_fwd_final.txt 2>&1
tail -n 1 gpurun_out/ncu_fwd_final.txt
