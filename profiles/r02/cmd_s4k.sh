timeout 300 python profiles/r02/c2_epi_ab.py "0 1 2" 2>&1 | tail -1
