for i in 1 2; do
echo base; DG_LIB=$PWD/profiles/r02/libdgmf_base.so timeout 200 python profiles/vcycle_once.py 2>&1 | grep "V-cycle"
echo new; timeout 200 python profiles/vcycle_once.py 2>&1 | grep "V-cycle"
done
timeout 600 python -m pytest tests/test_gpu_mg.py -x -q 2>&1 | tail -1
