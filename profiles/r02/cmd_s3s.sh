timeout 1200 python -m pytest tests/test_gpu_laplace.py tests/test_gpu_slab.py tests/test_gpu_c2.py tests/test_gpu_mg.py tests/test_gpu_stepper.py -x -q 2>&1 | tail -2
timeout 200 python profiles/r02/vmult_ab.py "128,4 64,4 96,4 48,4" "0:0 8:3" 2>&1 | tail -1
timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep -v Warn
timeout 300 python profiles/r02/slab_parts.py 2>&1 | tail -4
