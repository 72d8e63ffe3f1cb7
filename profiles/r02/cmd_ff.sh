python profiles/r02/vec_once.py && \
ncu --set full --import-source on --clock-control none -k regex:"vl_apply|vl_trace|vpcg_update" -c 4 -o gpurun_out/r2ff_vec python profiles/r02/vec_once.py > gpurun_out/r2ff_ncu.log 2>&1; tail -3 gpurun_out/r2ff_ncu.log
python -m pytest tests/test_gpu_mg.py tests/test_gpu_laplace.py -x -q 2>&1 | tail -2
python profiles/r02/c4_prof.py > gpurun_out/c4_prof4.log 2>&1; head -5 gpurun_out/c4_prof4.log
