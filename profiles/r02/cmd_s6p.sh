DG_EPI_CFG=8 timeout 600 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -2
for i in 1 2; do
echo default; timeout 300 python profiles/cg_profile.py 2>&1 | tail -1
echo fsd; DG_EPI_CFG=8 timeout 300 python profiles/cg_profile.py 2>&1 | tail -1
done
