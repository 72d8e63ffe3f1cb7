python profiles/r02/vec_once.py && \
ncu --set full --import-source on --clock-control none -k regex:"vl_apply|vl_trace|vpcg_update" -c 4 -o gpurun_out/r2qq_vec python profiles/r02/vec_once.py > gpurun_out/r2qq_ncu.log 2>&1; tail -1 gpurun_out/r2qq_ncu.log
