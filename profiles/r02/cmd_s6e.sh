for i in 1 2; do
for cfg in 0 5 6 7 2; do
echo cfg $cfg; DG_EPI_CFG=$cfg timeout 300 python profiles/cg_profile.py 2>&1 | tail -1
done
done
