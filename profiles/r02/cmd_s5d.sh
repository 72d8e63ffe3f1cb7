timeout 1200 python -m pytest tests/test_gpu_laplace.py tests/test_gpu_slab.py tests/test_gpu_c2.py tests/test_gpu_mg.py -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
