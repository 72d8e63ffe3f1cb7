timeout 300 python profiles/r02/slab_tiles.py "0" 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_slab.py tests/test_gpu_laplace.py -x -q -k "slab" 2>&1 | tail -2
