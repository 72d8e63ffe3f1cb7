timeout 1200 python -m pytest tests/test_gpu_laplace.py tests/test_gpu_mg.py tests/test_gpu_c2.py tests/test_gpu_stepper.py tests/test_gpu_slab.py -x -q 2>&1 | tail -2
echo base; DG_LIB=$PWD/profiles/r02/libdgmf_base.so timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep -v Warn
echo new; timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep -v Warn
