export DG_LAP_VARIANT=7
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_laplace.py -k "3d or multibrick or config1 or slab or periodic or host_buffer" > gpurun_out/r2g_pytest.log 2>&1; tail -2 gpurun_out/r2g_pytest.log
for cfg in 0 1 2; do DG_L7CFG=$cfg timeout 300 python profiles/r02/vmult_ab.py 128,4 64,4 64,3 96,3 > gpurun_out/r2g_ab7_$cfg.log 2>&1; done
cat gpurun_out/r2g_ab7_*.log
python profiles/r02/one_vmult.py 128 4 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:laplace7 -s 1 -c 1 -o gpurun_out/r2g_l7q4 python profiles/r02/one_vmult.py 128 4 > gpurun_out/r2g_ncu.log 2>&1; tail -1 gpurun_out/r2g_ncu.log
