for i in 1 2; do
echo base; DG_LIB=$PWD/profiles/r02/libdgmf_base.so timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep brick
echo new; timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep brick
done
