python -m pytest tests/test_gpu_laplace.py -q -x -k "chebyshev" 2>&1 | tail -2
python profiles/r02/cheb_time.py 2>&1 | grep brick; DG_EPI_V4=1 python profiles/r02/cheb_time.py 2>&1 | grep brick
python -m pytest tests/test_gpu_mg.py tests/test_gpu_stepper.py -q -x 2>&1 | tail -2
python profiles/r02/c4_prof.py > gpurun_out/c4_prof10.log 2>&1; sed -n 3,5p gpurun_out/c4_prof10.log; grep "laplace7\|total" gpurun_out/c4_prof10.log
