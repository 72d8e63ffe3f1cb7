timeout 200 python profiles/r02/vmult_ab.py "64,5 48,5" "0:0 8:0 7:1" 2>&1 | tail -1
timeout 200 python profiles/r02/vmult_ab.py "64,3 96,3" "0:0 8:0 8:1 8:2 7:1 7:2" 2>&1 | tail -1
