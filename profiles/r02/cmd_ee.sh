python -m pytest tests/test_gpu_mg.py tests/test_gpu_stepper.py -x -q > gpurun_out/r2ee_tests.log 2>&1; tail -3 gpurun_out/r2ee_tests.log
python profiles/r02/small_ab.py 2>&1 | tail -8
python profiles/r02/c4_prof.py > gpurun_out/c4_prof3.log 2>&1; head -5 gpurun_out/c4_prof3.log; grep "dense\|coarse" gpurun_out/c4_prof3.log
