for i in 1 2; do
timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep -v Warn
DG_EPI_COL=1 timeout 200 python profiles/r02/cheb_time.py 2>&1 | grep -v Warn
done
B="python bench.py --steps 3 --warmup 3 --no-cg --no-step --no-e2e --no-cpu"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3n_launches.csv $B > gpurun_out/s3n_ncu_launch.log 2>&1; tail -1 gpurun_out/s3n_ncu_launch.log
