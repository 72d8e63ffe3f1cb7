timeout 900 python profiles/r02/chunk_occ_ab.py 2>&1 | tail -9
