for i in 1 2; do
echo base; DG_LIB=$PWD/profiles/r02/libdgmf_base.so timeout 100 python profiles/r02/c3_ab.py 0 2>&1 | tail -1
echo new; timeout 100 python profiles/r02/c3_ab.py 0 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_vecops.py tests/test_gpu_rhs.py tests/test_gpu_stepper.py -x -q 2>&1 | tail -2
