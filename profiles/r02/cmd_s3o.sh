timeout 900 python -m pytest tests/test_gpu_laplace.py tests/test_gpu_c2.py tests/test_gpu_mg.py -x -q 2>&1 | tail -3
timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep -v Warn
