timeout 300 python profiles/r02/vmult_ab.py "128,4 64,4 96,4" "0:0 8:7" 2>&1 | tail -1
