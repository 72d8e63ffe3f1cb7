for i in 1 2; do
DG_LIB=$PWD/profiles/r02/libdgmf_base.so timeout 100 python profiles/r02/c3_ab.py 0 2>&1 | tail -1
timeout 100 python profiles/r02/c3_ab.py 0 2>&1 | tail -1
done
