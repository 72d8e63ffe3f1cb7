python profiles/r02/cheb_time.py 2>&1 | grep DG_EXP
python profiles/r02/cg_c5.py 2>&1 | tail -1
python -m pytest tests/test_gpu_laplace.py tests/test_gpu_mg.py tests/test_gpu_slab.py tests/test_gpu_c2.py tests/test_gpu_rhs.py -x -q 2>&1 | tail -2
