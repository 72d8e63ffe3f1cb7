python profiles/r02/c3_ab.py 0,1,2,3,5 2>&1 | tail -6
python -m pytest tests/test_gpu_vecops.py -x -q 2>&1 | tail -2
