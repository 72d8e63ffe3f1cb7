timeout 600 python -m pytest tests/test_gpu_slab.py -x -q 2>&1 | tail -3
echo fused; timeout 300 python profiles/r02/cg_dots_ab.py 2>&1 | tail -3
echo unfused; DG_NO_DOTS_FUSED=1 timeout 300 python profiles/r02/cg_dots_ab.py 2>&1 | tail -3
