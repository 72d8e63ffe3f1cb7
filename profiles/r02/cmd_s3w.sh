for i in 1 2; do
DG_LIB=$PWD/profiles/r02/libdgmf_base.so timeout 200 python profiles/r02/vmult_ab.py "64,3 96,3 64,5 48,5" "0:0" 2>&1 | tail -1
timeout 200 python profiles/r02/vmult_ab.py "64,3 96,3 64,5 48,5" "0:0" 2>&1 | tail -1
done
