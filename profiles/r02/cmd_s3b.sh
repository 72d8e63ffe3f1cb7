timeout 100 python profiles/r02/vmult_ab.py "128,4" "8:0 8:14" 2>&1 | tail -2
timeout 100 python profiles/r02/vmult_ab.py "128,4" "8:0 8:11" 2>&1 | tail -2
