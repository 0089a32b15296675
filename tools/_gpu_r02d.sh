# backward variants A/B at C4 + correctness of the default (moments) sweep
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --ignore=tests/test_scale_parity_gpu.py > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
for v in default bwd9 bwdmb10 bwdskip bwdskipmb10 coefldc; do
  if [ $v = default ]; then L=""; else L=paper_2509_15645_b200/_build/var_$v/libgss_b200.so; fi
  GSS_LIB=$L timeout 600 python tools/time_render.py 40000000 3840 2160 3 > gpurun_out/ab_$v.txt 2>&1
  tail -1 gpurun_out/ab_$v.txt
done
