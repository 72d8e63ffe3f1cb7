python -m pytest tests/test_gpu_vpcg.py tests/test_gpu_stepper.py -x -q 2>&1 | tail -2
python profiles/r02/vec_time.py 2>&1 | tail -4
python profiles/r02/c4_prof.py > gpurun_out/c4_prof6.log 2>&1; head -5 gpurun_out/c4_prof6.log
