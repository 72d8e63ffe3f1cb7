python profiles/r02/c3_ab.py 1,0 2>&1 | tail -3
python -m pytest tests/test_gpu_vecops.py tests/test_gpu_rhs.py tests/test_gpu_stepper.py -x -q 2>&1 | tail -2
