timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_abi.py -x -q 2>&1 | tail -15
