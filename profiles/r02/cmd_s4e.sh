timeout 300 python profiles/r02/c4_prof.py > gpurun_out/s4e_c4prof.log 2>&1; head -60 gpurun_out/s4e_c4prof.log
