set -x
B="python bench.py --steps 3 --warmup 3 --no-cg --no-step --no-e2e --no-cpu"
$B > gpurun_out/r2t_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:laplace7 -s 3 -c 1 -o gpurun_out/r2t_full $B > gpurun_out/r2t_ncu_full.log 2>&1
$B > gpurun_out/r2t_plain2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_launches.csv $B > gpurun_out/r2t_ncu_launch.log 2>&1
tail -2 gpurun_out/r2t_ncu_full.log
