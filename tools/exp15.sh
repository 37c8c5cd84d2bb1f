timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -m gpu -x 2>&1 | tail -2
bash tools/exp13.sh
