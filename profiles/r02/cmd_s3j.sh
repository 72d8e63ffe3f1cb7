timeout 900 python -m pytest tests/test_gpu_laplace.py tests/test_gpu_slab.py tests/test_gpu_mg.py tests/test_gpu_stepper.py -x -q 2>&1 | tail -2
timeout 200 python profiles/r02/vmult_ab.py "64,3 64,4 64,5" "0:0" 2>&1 | tail -1
