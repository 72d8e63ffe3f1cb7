timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_laplace.py tests/test_gpu_mg.py -x -q 2>&1 | tail -3
for i in 1 2; do
echo dotS; timeout 300 python profiles/cg_profile.py 2>&1 | tail -1
echo coop; DG_EPI_CFG=3 timeout 300 python profiles/cg_profile.py 2>&1 | tail -1
done
