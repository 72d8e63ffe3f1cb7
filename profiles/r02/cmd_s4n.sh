timeout 900 python -m pytest tests/test_gpu_vecops.py tests/test_gpu_rhs.py tests/test_gpu_stepper.py -x -q 2>&1 | tail -2
