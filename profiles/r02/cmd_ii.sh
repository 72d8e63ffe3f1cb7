python -m pytest tests/test_gpu_vpcg.py tests/test_gpu_stepper.py tests/test_gpu_vecops.py -x -q 2>&1 | tail -3
python profiles/r02/vec_time.py 2>&1 | tail -4
DG_PCG_NO_GRAPH=1 python profiles/r02/vec_time.py 2>&1 | tail -2
python profiles/r02/c4_prof.py > gpurun_out/c4_prof5.log 2>&1; head -5 gpurun_out/c4_prof5.log; sed -n 8,30p gpurun_out/c4_prof5.log
