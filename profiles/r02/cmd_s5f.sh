for i in 1 2; do
echo base; DG_LIB=$PWD/profiles/r02/libdgmf_base.so timeout 200 python profiles/r02/vmult_ab.py "128,4 96,4" "0:0" 2>&1 | tail -1
echo new; timeout 200 python profiles/r02/vmult_ab.py "128,4 96,4" "0:0" 2>&1 | tail -1
done
