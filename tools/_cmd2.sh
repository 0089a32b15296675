export GSS_PARITY_OUT=$PWD/gpurun_out/parity.json
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --ignore=tests/test_scale_parity_gpu.py 2>&1 | tail -5
timeout 2400 python -m pytest tests/test_scale_parity_gpu.py -q -m gpu --durations=10 2>&1 | tail -30
