timeout 1200 python -m pytest tests/test_gpu_laplace.py tests/test_gpu_slab.py tests/test_gpu_c2.py -x -q 2>&1 | tail -2
