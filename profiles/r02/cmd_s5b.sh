timeout 200 python profiles/r02/pcie_bw.py 2>&1 | tail -2
timeout 300 python profiles/e2e_chunks.py 2>&1 | tail -7
