python profiles/r02/vec_time.py 2>&1 | tail -5
python -m pytest tests/test_gpu_vecops.py tests/test_gpu_vpcg.py tests/test_gpu_stepper.py tests/test_gpu_mg.py -x -q 2>&1 | tail -2
