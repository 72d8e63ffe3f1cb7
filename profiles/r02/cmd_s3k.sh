timeout 200 python profiles/r02/vmult_ab.py "64,5 48,5" "0:0 7:4 7:5" 2>&1 | tail -1
