# sweep: exp factor folded into a scaled conic (GSS_BWD_KFOLD) and 10 CTAs/SM at the new register count: parity + same-box A/B
set -x
mkdir -p gpurun_out
B=paper_2509_15645_b200/_build
GSS_LIB=$B/var_kf1/libgss_b200.so timeout 1200 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py "tests/test_scale_parity_gpu.py::test_c4_strip_forward_backward_vs_reference" "tests/test_scale_parity_gpu.py::test_c2_view_forward_backward_vs_reference" -x -q > gpurun_out/pytest_ba.txt 2>&1; tail -n 3 gpurun_out/pytest_ba.txt
for i in 1 2; do
  for v in default kf1 m10; do
    if [ $v = default ]; then L=; else L=$B/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 600 python tools/time_render.py 40000000 3840 2160 2 > gpurun_out/tr_ba_$v$i.txt 2>&1; echo "$v $(grep 'cam 7' gpurun_out/tr_ba_$v$i.txt)" >> gpurun_out/tr_ba.txt
  done
done
cat gpurun_out/tr_ba.txt
for i in 1 2; do
  for v in default kf1; do
    if [ $v = default ]; then L=; else L=$B/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_ba_$v$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_ba_$v$i.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_ba.txt
  done
done
cat gpurun_out/ab_ba.txt
