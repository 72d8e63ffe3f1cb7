for i in 1 2; do
echo list; timeout 300 python profiles/cg_profile.py 2>&1 | tail -2
echo wave; DG_CHUNK_MODEL=0 timeout 300 python profiles/cg_profile.py 2>&1 | tail -2
done
