timeout 200 python profiles/r02/vmult_ab.py "64,5 48,5" "7:2 7:3 7:4" 2>&1 | tail -1
timeout 200 python profiles/r02/vmult_ab.py "64,3 96,3" "0:0 7:3 7:4" 2>&1 | tail -1
