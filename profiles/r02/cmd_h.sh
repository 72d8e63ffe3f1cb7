export DG_LAP_VARIANT=7
for cfg in 0 1 2 3; do DG_L7CFG=$cfg timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_laplace.py -k "3d or multibrick or config1 or slab or periodic or host_buffer" > gpurun_out/r2h_pytest_$cfg.log 2>&1; tail -1 gpurun_out/r2h_pytest_$cfg.log; done
for cfg in 0 1 2 3; do DG_L7CFG=$cfg timeout 300 python profiles/r02/vmult_ab.py 128,4 64,4 64,3 96,3 > gpurun_out/r2h_ab7_$cfg.log 2>&1; done
cat gpurun_out/r2h_ab7_*.log
