python -m pytest tests/test_gpu_laplace.py tests/test_gpu_mg.py tests/test_gpu_stepper.py tests/test_gpu_slab.py -x -q > gpurun_out/r2dd_tests.log 2>&1; tail -5 gpurun_out/r2dd_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -6
python profiles/r02/c4_prof.py > gpurun_out/c4_prof2.log 2>&1; head -5 gpurun_out/c4_prof2.log; grep -v "^ *[0-9.]*% *[0-9.]* us *[0-9]* x *[0-9.]* us  ([0-9]*, 1, 1) *dg::laplace_vmult" gpurun_out/c4_prof2.log | sed -n 6,40p
